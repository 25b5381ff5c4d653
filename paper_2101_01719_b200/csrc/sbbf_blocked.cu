// sbbf_blocked.cu — multisplit partitions: the L2-blocked insert/lookup for
// filters larger than L2, and the shard routing of the multi-GPU path.
//
// A random 32-byte probe that misses L2 costs a full DRAM line fill
// (ncu: ~117 B of DRAM per key on a 1 GiB filter) and the HBM random-sector
// rate tops out at 37-43 G/s whatever the access path (LSU, TMA, gather4;
// profiles/r1_microbench_*.log). The blocked path trades that for streaming:
//
//   1. chunk_scatter: every 4096-key chunk of the batch is rewritten
//      bucket-major (bucket = filter slice of ~32 MiB) inside its own region,
//      with 16-bit bucket offsets per chunk: one read, coalesced writes, no
//      count pass;
//   2. inserts — segment_kernel: bucket by bucket over every chunk's run of
//      that bucket; the keys in flight share one slice, so their atomics are
//      served by L2 and each filter line comes from HBM about once per call;
//   3. lookups — sweep_find_kernel (the fused sweep): the partition stores
//      packed slots (slice-relative block, source position, low hash bits)
//      and one persistent, slice-paced grid probes them and sets each hit's
//      bit at its source position in per-chunk result rows in shared memory,
//      written out as the caller's bits or bytes. Maps whose slices exceed
//      2^20 blocks, and the multi-region calls of the sharded layer, keep the
//      older form: segment_kernel storing an answer byte per routed slot,
//      then unpermute_kernel (each chunk's answers back to source order
//      through shared memory).
//
// Per-key HBM traffic of a config-4 lookup ~ 8 + 8 (scatter) + 8 (sweep) +
// filter_bytes x ~1.3 / round keys + 1/8 (ncu: profiles/traffic.json); the
// unfused form adds 2 + 2 (positions) + 1 + 1 (answer bytes).
//
// The shard routing (shard_partition / route_partition) needs one
// bucket-major layout over the whole batch instead: bucket_count ->
// bucket_scan (per-CTA bases) -> bucket_scatter, which can also write each
// destination's run straight into a peer GPU's window (sbbf_route.cu).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <new>
#include <tuple>
#include <vector>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

constexpr int kBlockedRoundLog2 = 28;  // keys per blocked round (~3 GB of scratch for lookups)
// SBBF_BLOCKED_ROUND_LOG2 overrides the round size (A/B only, 24..31).
uint64_t blocked_round() {
  static const uint64_t v = [] {
    const char* e = getenv("SBBF_BLOCKED_ROUND_LOG2");
    const int x = e ? atoi(e) : 0;
    return uint64_t{1} << (x >= 24 && x <= 31 ? x : kBlockedRoundLog2);
  }();
  return v;
}

// ---------------------------------------------------------------------------
// per-kernel live timing for bench.py (sbbf_bench_kernel_timing / _times)
// ---------------------------------------------------------------------------
// When enabled, every blocked-path launch group is bracketed by two CUDA
// events on its stream; sbbf_bench_kernel_times() synchronises them and sums
// the durations per kind. Off by default (no events are recorded).
enum KernelKind { kKPartition = 0, kKProbe = 1, kKInsertSweep = 2, kKUnpermute = 3, kKTile = 4, kKNum = 5 };

struct KTimer {
  std::mutex mu;
  std::atomic<bool> on{false};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
  double ms[kKNum] = {};
  uint64_t n[kKNum] = {};
};
KTimer& ktimer() {
  static KTimer* t = new KTimer;  // never destroyed: events may outlive static teardown order
  return *t;
}

class KTime {
 public:
  KTime(int kind, cudaStream_t s) : kind_(kind), s_(s) {
    KTimer& t = ktimer();
    if (!t.on.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lock(t.mu);
    if (t.pool.empty()) {
      cudaEvent_t a = nullptr, b = nullptr;
      if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      t.pool.emplace_back(a, b);
    }
    ev_ = t.pool.back();
    t.pool.pop_back();
    active_ = cudaEventRecord(ev_.first, s_) == cudaSuccess;
  }
  ~KTime() {
    if (!active_) return;
    KTimer& t = ktimer();
    cudaEventRecord(ev_.second, s_);
    std::lock_guard<std::mutex> lock(t.mu);
    t.pending.emplace_back(kind_, ev_.first, ev_.second);
  }

 private:
  int kind_;
  cudaStream_t s_;
  std::pair<cudaEvent_t, cudaEvent_t> ev_{nullptr, nullptr};
  bool active_ = false;
};

// ---------------------------------------------------------------------------
// bucket partition
// ---------------------------------------------------------------------------
// Bucket of a key = its local block scaled to [0, S) by a 32.32 fixed-point
// multiply: monotone in the block, so bucket k is a contiguous block range of
// ~nb/S blocks (neighbouring buckets may share a boundary block — harmless,
// each key is still handled on its own). S <= 64 for the whole-batch partition, <= 128 for the chunk-local one.
//
// Ranking inside a warp is a ballot "multisplit": for a BITS-bit bucket id,
// BITS ballots give every lane the mask of lanes holding its bucket (AND of
// ballot or ~ballot per bit). Per-warp running counts live in registers —
// lane l owns buckets l and l+32 — so there are no per-key shared-memory
// atomics (~2 cycles per lane on this part) and no __match_any_sync (which
// measured slower still: profiles/r1_blocked_partition.md).
constexpr int kPartThreads = 512;
constexpr int kPartMinBlocks = 2;
constexpr int kPartWarps = kPartThreads / 32;
constexpr int kPartPerThread = 8;
constexpr uint64_t kPartChunk = kPartThreads * kPartPerThread;
constexpr int kMaxBuckets = 64;     // whole-batch partition (shard routing, super-slices)
constexpr int kMaxBits = 6;
constexpr int kChunkBuckets = 128;  // chunk-local partition (blocked path): up to 128 slices
constexpr int kChunkBits = 8;  // bal[] capacity: chunk-local ids use <= 7 bits, tile ids 8
// buckets each lane owns (lane + 32 i) for BITS-bit bucket ids
template <int BITS>
constexpr int owned() { return BITS > 5 ? 1 << (BITS - 5) : 1; }

struct BucketMap {
  uint64_t nb_global, first, nb_local, mult;  // mult = floor(S * 2^32 / nb_local)
  uint32_t S, bits;
  const uint64_t* bounds;  // optional exact bucket starts (local block ids), S entries
  bool top_bits;           // whole filter, S = 2^bits: bucket = top bits of the hash
  // Packed staging (fused lookups, chunk-local partition only): a slot holds
  // (block offset inside its slice) << 44 | (source position in the chunk) << 32
  // | the hash's low 32 bits — all the probe and the answer need — instead of
  // the hash, so no position array is written. pack_shift (top_bits maps) is
  // 64 - log2(blocks per slice); `sentinel` marks keys outside the shard.
  uint32_t pack = 0, pack_shift = 0, sentinel = 0;
};

constexpr int kPackOffBits = 20;                           // slices of <= 2^20 blocks (32 MiB)
constexpr uint32_t kPackForeign = (1u << kPackOffBits) - 1;  // offset of a key outside the shard (sentinel maps)

// First local block of bucket q under bucket_of's fixed-point map:
// q = floor(b * mult / 2^32) (clamped to S - 1) is monotone in b, so bucket q
// starts at ceil(q * 2^32 / mult).
__host__ __device__ __forceinline__ uint64_t bucket_start(uint64_t q, uint64_t mult) {
  return ((q << 32) + mult - 1) / mult;
}

// kTop: the map is a whole filter split into S = 2^bits slices. block_index
// is monotone in the hash, so the hash's top bits split the filter into S
// contiguous block ranges without any 64-bit multiply.
template <bool kTop>
__device__ __forceinline__ uint32_t bucket_of(uint64_t h, const BucketMap& bm) {
  if constexpr (kTop) return static_cast<uint32_t>(h >> (64 - bm.bits));
  uint64_t b = dev::block_index(h, bm.nb_global) - bm.first;
  b = b < bm.nb_local ? b : 0;
  uint64_t q = b * bm.mult >> 32;
  q = q < bm.S ? q : bm.S - 1;
  if (bm.bounds) {
    // exact ranges (multi-GPU shards: [floor(rB/P), floor((r+1)B/P))): the
    // fixed-point estimate is within one of the owner
    while (q + 1 < bm.S && b >= __ldg(bm.bounds + q + 1)) ++q;
    while (q > 0 && b < __ldg(bm.bounds + q)) --q;
  }
  return static_cast<uint32_t>(q);
}

// One ballot per bucket-id bit. Written in PTX so that each bit is a single
// predicate-producing LOP3 feeding the VOTE (the C++ form compiled to a
// shift, a mask and a 64-bit compare per bit).
template <int BITS>
__device__ __forceinline__ void bit_ballots(uint32_t bk, uint32_t (&bal)[kChunkBits]) {
#pragma unroll
  for (int k = 0; k < BITS; ++k)
    asm("{ .reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 %0, p, 0xffffffff; }"
        : "=r"(bal[k])
        : "r"(bk), "r"(1u << k));
}

__device__ __forceinline__ uint32_t flip(uint32_t v, int k) { return ((v >> k) & 1u) - 1u; }

// Per-lane flip masks of the buckets lane l owns (l + 32 i), hoisted out of
// the key loops: bits 0..4 are shared by all of them.
struct OwnerMasks {
  uint32_t f[5];
  __device__ __forceinline__ explicit OwnerMasks(uint32_t lane) {
#pragma unroll
    for (int k = 0; k < 5; ++k) f[k] = flip(lane, k);
  }
};

// m[i] = the lanes of this warp step whose key is in bucket lane + 32 i.
template <int BITS>
__device__ __forceinline__ void owner_masks(const OwnerMasks& om, const uint32_t (&bal)[kChunkBits], uint32_t active,
                                            uint32_t (&m)[owned<BITS>()]) {
  constexpr int kLow = BITS < 5 ? BITS : 5;
  uint32_t base = active;
#pragma unroll
  for (int k = 0; k < kLow; ++k) base &= bal[k] ^ om.f[k];
#pragma unroll
  for (int i = 0; i < owned<BITS>(); ++i) {
    uint32_t x = base;
    if constexpr (BITS > 5) x &= (i & 1) ? bal[5] : ~bal[5];
    if constexpr (BITS > 6) x &= (i & 2) ? bal[6] : ~bal[6];
    if constexpr (BITS > 7) x &= (i & 4) ? bal[7] : ~bal[7];
    m[i] = x;
  }
}

// Add this warp step's counts of the lane's owned buckets to c[].
template <int BITS>
__device__ __forceinline__ void owner_counts(const OwnerMasks& om, const uint32_t (&bal)[kChunkBits], uint32_t active,
                                             uint32_t (&c)[owned<BITS>()]) {
  uint32_t m[owned<BITS>()];
  owner_masks<BITS>(om, bal, active, m);
#pragma unroll
  for (int i = 0; i < owned<BITS>(); ++i) c[i] += __popc(m[i]);
}

// One warp step over 32 keys: rank of each lane inside its bucket group and
// the per-bucket counts added to the lane-owned counters c[i] (bucket =
// lane + 32 i). Each lane first forms the masks of lanes holding the buckets
// it owns (BITS LOP3s against its precomputed flip masks); a key's peer mask
// and prior count then come from its bucket's owner lane by shuffle, instead
// of every lane rebuilding its own bucket's mask bit by bit.
template <int BITS>
__device__ __forceinline__ uint32_t warp_rank(uint32_t bk, bool valid, uint32_t lane, const OwnerMasks& om,
                                              uint32_t (&c)[owned<BITS>()]) {
  const uint32_t active = __ballot_sync(0xffffffffu, valid);
  uint32_t bal[kChunkBits];
  bit_ballots<BITS>(bk, bal);
  uint32_t m[owned<BITS>()];
  owner_masks<BITS>(om, bal, active, m);
  const uint32_t src = bk & 31, hi = bk >> 5;
  uint32_t peers = 0, prior = 0;
#pragma unroll
  for (int i = 0; i < owned<BITS>(); ++i) {
    const uint32_t p = __shfl_sync(0xffffffffu, m[i], src);
    const uint32_t q = __shfl_sync(0xffffffffu, c[i], src);
    if (owned<BITS>() == 1 || hi == static_cast<uint32_t>(i)) {
      peers = p;
      prior = q;
    }
  }
#pragma unroll
  for (int i = 0; i < owned<BITS>(); ++i) c[i] += __popc(m[i]);
  return prior + __popc(peers & ((1u << lane) - 1u));
}

// Slot of each key in the chunk's bucket-major smem staging: lane l fetches
// its warp's base of its owned buckets once (bucket offset + this warp's
// prefix), and each key takes its bucket's base by shuffle — no dependent
// per-key shared-memory loads (they were ~30 % of chunk_scatter's stalls).
template <int BITS>
__device__ __forceinline__ uint32_t slot_base(uint32_t bk, const uint32_t (&base)[owned<BITS>()]) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < owned<BITS>(); ++i) {
    const uint32_t b = __shfl_sync(0xffffffffu, base[i], bk & 31);
    if (owned<BITS>() == 1 || (bk >> 5) == static_cast<uint32_t>(i)) r = b;
  }
  return r;
}

// The value a chunk slot stores: the hash, or (packed maps) what the fused
// lookup sweep needs of it. `starts` = the CTA's table of bucket starts
// (maps without top_bits).
template <bool kTop>
__device__ __forceinline__ uint64_t slot_value(uint64_t h, uint32_t bk, uint32_t pos, const BucketMap& bm,
                                               const uint64_t* starts) {
  if (!bm.pack) return h;
  uint64_t off;
  if constexpr (kTop) {
    // power-of-two filters: a bit field of the hash; otherwise bucket bk's first
    // block is mulhi(bk << (64 - bits), nb) = (bk * nb) >> bits
    off = bm.pack_shift ? (h << bm.bits) >> bm.pack_shift
                        : dev::block_index(h, bm.nb_global) - ((static_cast<uint64_t>(bk) * bm.nb_global) >> bm.bits);
    SBBF_DCHECK(off < (1u << kPackOffBits));
  } else {
    const uint64_t b = dev::block_index(h, bm.nb_global) - bm.first;
    off = b < bm.nb_local ? b - starts[bk] : kPackForeign;
    SBBF_DCHECK(b >= bm.nb_local || (b >= starts[bk] && b - starts[bk] < (1u << kPackOffBits) - bm.sentinel));
  }
  return off << 44 | static_cast<uint64_t>(pos) << 32 | static_cast<uint32_t>(h);
}

// Bucket starts of a packed map without top_bits, into shared memory.
template <bool kTop>
__device__ __forceinline__ void fill_starts(const BucketMap& bm, uint64_t* starts) {
  if constexpr (!kTop) {
    if (bm.pack)
      for (uint32_t q = threadIdx.x; q < bm.S; q += blockDim.x) starts[q] = bucket_start(q, bm.mult);
  }
}

// Both passes give CTA c the same contiguous run of chunks, so the count
// pass can hand each CTA exact per-bucket output offsets (after a tiny scan)
// and the scatter pass needs no global atomics on its critical path.
__device__ __forceinline__ void cta_chunk_range(uint64_t n, uint64_t& c0, uint64_t& c1) {
  const uint64_t nchunks = (n + kPartChunk - 1) / kPartChunk;
  const uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  c0 = static_cast<uint64_t>(blockIdx.x) * per;
  c1 = c0 + per < nchunks ? c0 + per : nchunks;
}

// Loads of one partition chunk (8 keys per thread, coalesced). Chunks entirely
// inside [0, n) skip the per-key bounds checks.
__device__ __forceinline__ void load_chunk(const uint64_t* __restrict__ hashes, uint64_t n, uint64_t ch,
                                           uint64_t pol, uint64_t (&dst)[kPartPerThread]) {
  const uint64_t base = ch * kPartChunk + threadIdx.x;
  if (base - threadIdx.x + kPartChunk <= n) {
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) dst[j] = dev::ld_stream_u64(hashes + base + j * kPartThreads, pol);
  } else {
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kPartThreads;
      dst[j] = i < n ? dev::ld_stream_u64(hashes + i, pol) : 0;
    }
  }
}

template <int BITS, bool kTop>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks) bucket_count_kernel(const uint64_t* __restrict__ hashes,
                                                                       uint64_t n, BucketMap bm,
                                                                       uint32_t* __restrict__ cta_hist) {
  __shared__ unsigned int cta[kMaxBuckets];
  const uint32_t lane = threadIdx.x & 31;
  const OwnerMasks om(lane);
  const uint64_t pol = dev::policy_evict_first();
  if (threadIdx.x < kMaxBuckets) cta[threadIdx.x] = 0;
  uint32_t c[owned<BITS>()] = {};
  uint64_t ch0, ch1;
  cta_chunk_range(n, ch0, ch1);
  // Software pipeline: the next chunk's loads are in flight while this
  // chunk's ballots run (the kernel is otherwise latency bound).
  uint64_t nxt[kPartPerThread];
  if (ch0 < ch1) load_chunk(hashes, n, ch0, pol, nxt);
  for (uint64_t ch = ch0; ch < ch1; ++ch) {
    uint64_t h[kPartPerThread];
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) h[j] = nxt[j];
    if (ch + 1 < ch1) load_chunk(hashes, n, ch + 1, pol, nxt);
    const uint64_t base = ch * kPartChunk;
    if (base + kPartChunk <= n) {
#pragma unroll
      for (int j = 0; j < kPartPerThread; ++j) {
        uint32_t bal[kChunkBits];
        bit_ballots<BITS>(bucket_of<kTop>(h[j], bm), bal);
        owner_counts<BITS>(om, bal, 0xffffffffu, c);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPartPerThread; ++j) {
        const uint64_t i = base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
        const uint32_t bk = i < n ? bucket_of<kTop>(h[j], bm) : 0u;
        const uint32_t active = __ballot_sync(0xffffffffu, i < n);
        uint32_t bal[kChunkBits];
        bit_ballots<BITS>(bk, bal);
        owner_counts<BITS>(om, bal, active, c);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < owned<BITS>(); ++i)
    if (lane + 32 * i < bm.S && c[i]) atomicAdd(&cta[lane + 32 * i], c[i]);
  __syncthreads();
  if (threadIdx.x < kMaxBuckets) cta_hist[static_cast<uint64_t>(blockIdx.x) * kMaxBuckets + threadIdx.x] = cta[threadIdx.x];
}

// counts[b] = total of bucket b; cta_base[c][b] = first output slot of CTA c's
// keys in bucket b (buckets are laid out in order, CTAs in order inside each).
__global__ void bucket_scan_kernel(const uint32_t* __restrict__ cta_hist, uint32_t ctas, uint32_t S,
                                   unsigned long long* __restrict__ counts,
                                   unsigned long long* __restrict__ cta_base) {
  __shared__ unsigned long long tot[kMaxBuckets];
  const uint32_t b = threadIdx.x;  // one thread per bucket
  unsigned long long t = 0;
  if (b < S)
    for (uint32_t c = 0; c < ctas; ++c) t += cta_hist[static_cast<uint64_t>(c) * kMaxBuckets + b];
  tot[b] = t;
  __syncthreads();
  if (b < S) {
    unsigned long long start = 0;
    for (uint32_t k = 0; k < b; ++k) start += tot[k];
    counts[b] = t;
    for (uint32_t c = 0; c < ctas; ++c) {
      cta_base[static_cast<uint64_t>(c) * kMaxBuckets + b] = start;
      start += cta_hist[static_cast<uint64_t>(c) * kMaxBuckets + b];
    }
  }
}

// Scatter through shared memory: each chunk is first placed bucket-major in
// smem (ballot ranks, no atomics), then copied out so that consecutive
// threads write consecutive slots of one bucket run — coalesced stores
// instead of one scattered 8-byte store per key.
struct ScatterSmem {
  uint64_t key[kPartChunk];
  uint32_t pos[kPartChunk];
  uint8_t bk[kPartChunk];
  uint32_t wcnt[kPartWarps][kMaxBuckets];  // per-warp counts -> exclusive prefix over warps
  uint32_t boff[kMaxBuckets];              // exclusive prefix over buckets (chunk-local)
  unsigned long long gbase[kMaxBuckets];   // global slot of this chunk's run, per bucket
  unsigned long long cursor[kMaxBuckets];  // this CTA's next slot per bucket
  unsigned long long bstart[kMaxBuckets];  // first slot of each bucket (routed mode)
  uint64_t* dst[kMaxBuckets];              // routed mode: bucket b's run goes to dst[b][slot - bstart[b]]
};

// Routed mode of the scatter (fused multi-GPU dispatch, sbbf_route.cu): the
// bucket-major run of bucket b is written straight into destination b's
// window — a peer GPU's receive buffer mapped over NVLink — instead of a
// local staging array, and block 0 publishes the per-bucket counts there.
struct RouteOut {
  uint64_t* const* dst = nullptr;                  // [S] window base for this source, per destination
  unsigned long long* const* count_dst = nullptr;  // [S] where destination b expects this source's count
};

template <int BITS, bool kTop>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks) bucket_scatter_kernel(
    const uint64_t* __restrict__ hashes, uint64_t n, BucketMap bm,
    const unsigned long long* __restrict__ cta_base, uint64_t* __restrict__ out, uint32_t* __restrict__ pos,
    RouteOut route = RouteOut{}, const unsigned long long* __restrict__ counts = nullptr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScatterSmem& sm = *reinterpret_cast<ScatterSmem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OwnerMasks om(lane);
  const uint64_t pol = dev::policy_evict_first();
  const bool routed = route.dst != nullptr;
  if (threadIdx.x < kMaxBuckets) {
    sm.cursor[threadIdx.x] = cta_base[static_cast<uint64_t>(blockIdx.x) * kMaxBuckets + threadIdx.x];
    if (routed) {
      const bool used = threadIdx.x < bm.S;
      sm.bstart[threadIdx.x] = cta_base[threadIdx.x];  // CTA 0's base = the bucket's first slot
      sm.dst[threadIdx.x] = used ? route.dst[threadIdx.x] : nullptr;
      // every destination learns how many keys this source sends it (zero included)
      if (blockIdx.x == 0 && used) *route.count_dst[threadIdx.x] = counts[threadIdx.x];
    }
  }
  uint64_t ch0, ch1;
  cta_chunk_range(n, ch0, ch1);
  for (uint64_t ch = ch0; ch < ch1; ++ch) {
    const uint64_t base = ch * kPartChunk;
    const uint32_t cnt = static_cast<uint32_t>(n - base < kPartChunk ? n - base : kPartChunk);
    uint64_t h[kPartPerThread];
    uint32_t bk[kPartPerThread], off[kPartPerThread];
    load_chunk(hashes, n, ch, pol, h);
    uint32_t c[owned<BITS>()] = {};
    if (cnt == kPartChunk) {
#pragma unroll
      for (int j = 0; j < kPartPerThread; ++j) {
        bk[j] = bucket_of<kTop>(h[j], bm);
        off[j] = warp_rank<BITS>(bk[j], true, lane, om, c);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPartPerThread; ++j) {
        const uint64_t i = base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
        const bool valid = i < n;
        bk[j] = valid ? bucket_of<kTop>(h[j], bm) : 0u;
        off[j] = warp_rank<BITS>(bk[j], valid, lane, om, c);
        if (!valid) bk[j] = 0xffffffffu;
      }
    }
#pragma unroll
    for (int i = 0; i < kMaxBuckets / 32; ++i) sm.wcnt[warp][lane + 32 * i] = i < owned<BITS>() ? c[i] : 0u;
    __syncthreads();
    if (warp == 0) {
      // bucket totals (lane owns buckets lane, lane+32), warp prefixes, a
      // warp-wide exclusive scan over the 64 buckets, and this CTA's own
      // cursors (no global atomics: offsets came from the count pass)
      uint32_t t0 = 0, t1 = 0;
#pragma unroll
      for (int w = 0; w < kPartWarps; ++w) {
        const uint32_t a = sm.wcnt[w][lane], b = sm.wcnt[w][lane + 32];
        sm.wcnt[w][lane] = t0;
        sm.wcnt[w][lane + 32] = t1;
        t0 += a;
        t1 += b;
      }
      uint32_t s0 = t0, s1 = t1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y0 = __shfl_up_sync(0xffffffffu, s0, d), y1 = __shfl_up_sync(0xffffffffu, s1, d);
        if (lane >= static_cast<uint32_t>(d)) {
          s0 += y0;
          s1 += y1;
        }
      }
      const uint32_t sum0 = __shfl_sync(0xffffffffu, s0, 31);
      sm.boff[lane] = s0 - t0;
      sm.boff[lane + 32] = sum0 + s1 - t1;
      sm.gbase[lane] = sm.cursor[lane];
      sm.gbase[lane + 32] = sm.cursor[lane + 32];
      sm.cursor[lane] += t0;
      sm.cursor[lane + 32] += t1;
    }
    __syncthreads();
    uint32_t sbase[owned<BITS>()];
#pragma unroll
    for (int i = 0; i < owned<BITS>(); ++i) sbase[i] = sm.boff[lane + 32 * i] + sm.wcnt[warp][lane + 32 * i];
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint32_t loc = slot_base<BITS>(bk[j], sbase) + off[j];
      if (bk[j] != 0xffffffffu) {
        sm.key[loc] = h[j];
        sm.pos[loc] = static_cast<uint32_t>(base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x);
        sm.bk[loc] = static_cast<uint8_t>(bk[j]);
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += kPartThreads) {
      const uint32_t b = sm.bk[i];
      const uint64_t slot = sm.gbase[b] + (i - sm.boff[b]);
      SBBF_DCHECK(b < bm.S && i >= sm.boff[b] && (routed || slot < n));
      if (routed)
        sm.dst[b][slot - sm.bstart[b]] = sm.key[i];  // consecutive threads -> consecutive peer slots
      else
        out[slot] = sm.key[i];
      if (pos) pos[slot] = sm.pos[i];
    }
    __syncthreads();
  }
  // peer stores are weakly ordered: make them visible system-wide before the
  // grid completes (the host then orders the owner's read behind a collective)
  if (routed) __threadfence_system();
}

BucketMap make_map(const Geom& g, uint32_t S) {
  BucketMap bm;
  bm.nb_global = g.nb_global;
  bm.first = g.first;
  bm.nb_local = g.nb_local;
  bm.S = S;
  bm.bits = 0;
  while ((1u << bm.bits) < S) ++bm.bits;
  if (bm.bits == 0) bm.bits = 1;  // a single bucket still needs a 1-bit id
  bm.mult = static_cast<uint64_t>((static_cast<unsigned __int128>(S) << 32) / g.nb_local);
  bm.bounds = nullptr;
  bm.top_bits = g.first == 0 && g.nb_local == g.nb_global && (1u << bm.bits) == S;
  return bm;
}

// Scratch comes from the stream-ordered pool; keep freed blocks cached in the
// pool (release threshold = max) so per-call allocations do not go back to
// the driver at every synchronisation.
void retain_pool() {
  static std::atomic<uint64_t> done{0};  // bit per device ordinal < 64
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  const uint64_t bit = uint64_t{1} << dev;
  if (done.load(std::memory_order_relaxed) & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~uint64_t{0};
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.fetch_or(bit, std::memory_order_relaxed);
}

template <int BITS, bool kTop>
cudaError_t bucket_partition_bits(uint64_t grid, const BucketMap& bm, const uint64_t* hashes, uint64_t m,
                                  uint64_t* d_counts, uint64_t* d_out, uint32_t* d_pos, cudaStream_t s,
                                  RouteOut route = RouteOut{}) {
  retain_pool();
  // per-CTA histograms and bases (grid x 64 entries) from the stream-ordered pool
  uint32_t* hist = nullptr;
  unsigned long long* bases = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&hist), grid * kMaxBuckets * sizeof(uint32_t), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&bases), grid * kMaxBuckets * sizeof(unsigned long long), s);
  static const cudaError_t attr = cudaFuncSetAttribute(
      bucket_scatter_kernel<BITS, kTop>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      static_cast<int>(sizeof(ScatterSmem)));
  if (e == cudaSuccess) e = attr;
  if (e == cudaSuccess) {
    note_launch();
    bucket_count_kernel<BITS, kTop><<<static_cast<unsigned>(grid), kPartThreads, 0, s>>>(hashes, m, bm, hist);
    note_launch();
    bucket_scan_kernel<<<1, kMaxBuckets, 0, s>>>(hist, static_cast<uint32_t>(grid), bm.S,
                                                 reinterpret_cast<unsigned long long*>(d_counts), bases);
    note_launch();
    bucket_scatter_kernel<BITS, kTop><<<static_cast<unsigned>(grid), kPartThreads, sizeof(ScatterSmem), s>>>(
        hashes, m, bm, bases, d_out, d_pos, route, reinterpret_cast<const unsigned long long*>(d_counts));
    e = cudaGetLastError();
  }
  if (hist) cudaFreeAsync(hist, s);
  if (bases) cudaFreeAsync(bases, s);
  return e;
}

// Group `m` keys by bucket: d_out (and d_pos) receive them bucket-major.
cudaError_t bucket_partition(const DeviceInfo& di, const Geom& g, uint32_t S, const uint64_t* hashes,
                             uint64_t m, uint64_t* d_counts, uint64_t* d_cursor, uint64_t* d_out,
                             uint32_t* d_pos, cudaStream_t s, const uint64_t* d_bounds = nullptr,
                             RouteOut route = RouteOut{}) {
  (void)d_cursor;
  BucketMap bm = make_map(g, S);
  bm.bounds = d_bounds;
  // exact shard ranges: top hash bits equal the owner only when B is a power of two
  if (d_bounds && (g.nb_global & (g.nb_global - 1)) != 0) bm.top_bits = false;
  // an empty batch still runs the (tiny) grid in routed mode: every destination
  // must receive this source's zero counts
  if (m == 0 && !route.dst) return cudaMemsetAsync(d_counts, 0, S * sizeof(uint64_t), s);
  const uint64_t grid = m ? grid_for(m, kPartChunk, di.sms, kPartMinBlocks) : 1;
  switch (bm.bits * 2 + (bm.top_bits ? 1 : 0)) {
#define SBBF_PART_CASE(B)                                                                                       \
  case 2 * B:                                                                                                   \
    return bucket_partition_bits<B, false>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);         \
  case 2 * B + 1:                                                                                               \
    return bucket_partition_bits<B, true>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    SBBF_PART_CASE(1)
    SBBF_PART_CASE(2)
    SBBF_PART_CASE(3)
    SBBF_PART_CASE(4)
    SBBF_PART_CASE(5)
    SBBF_PART_CASE(6)
#undef SBBF_PART_CASE
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// chunk-local blocked path (filters beyond L2)
// ---------------------------------------------------------------------------
// chunk_scatter: every kPartChunk-key chunk of the batch is rewritten
// bucket-major INSIDE ITS OWN REGION [ch*K, ch*K + cnt): one read of the
// keys, fully coalesced writes, no count pass, no scan, no global atomics.
// Per chunk it records the bucket offsets boffs[ch][0..S] (16-bit) and, for
// lookups, each slot's 16-bit source position inside the chunk.
struct ChunkSmem {
  uint64_t key[kPartChunk];
  alignas(16) uint16_t pos[kPartChunk];
  uint32_t wcnt[kPartWarps][kChunkBuckets];
  uint32_t boff[kChunkBuckets + 1];
};
constexpr int kBoffStride = kChunkBuckets + 1;

template <int BITS, bool kTop>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks)
    chunk_scatter_kernel(const uint64_t* __restrict__ hashes, uint64_t n, BucketMap bm, uint64_t* __restrict__ out,
                         uint16_t* __restrict__ pos16, uint16_t* __restrict__ boffs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChunkSmem& sm = *reinterpret_cast<ChunkSmem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OwnerMasks om(lane);
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t nchunks = (n + kPartChunk - 1) / kPartChunk;
  // packed maps write no positions: the array's space holds the bucket starts
  uint64_t* const starts = reinterpret_cast<uint64_t*>(sm.pos);
  fill_starts<kTop>(bm, starts);
  if (bm.pack) pos16 = nullptr;
  for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const uint64_t base = ch * kPartChunk;
    const uint32_t cnt = static_cast<uint32_t>(n - base < kPartChunk ? n - base : kPartChunk);
    uint64_t h[kPartPerThread];
    uint32_t bk[kPartPerThread], off[kPartPerThread];
    load_chunk(hashes, n, ch, pol, h);
    uint32_t c[owned<BITS>()] = {};
    if (cnt == kPartChunk) {
#pragma unroll
      for (int j = 0; j < kPartPerThread; ++j) {
        bk[j] = bucket_of<kTop>(h[j], bm);
        off[j] = warp_rank<BITS>(bk[j], true, lane, om, c);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPartPerThread; ++j) {
        const bool valid = j * kPartThreads + threadIdx.x < cnt;
        bk[j] = valid ? bucket_of<kTop>(h[j], bm) : 0u;
        off[j] = warp_rank<BITS>(bk[j], valid, lane, om, c);
        if (!valid) bk[j] = 0xffffffffu;
      }
    }
#pragma unroll
    for (int i = 0; i < kChunkBuckets / 32; ++i) sm.wcnt[warp][lane + 32 * i] = i < owned<BITS>() ? c[i] : 0u;
    __syncthreads();
    if (warp == 0) {
      // per-bucket totals over the warps (lane owns buckets lane + 32 i),
      // exclusive prefixes over warps and over buckets
      constexpr int kO = owned<BITS>();
      uint32_t t[kO] = {};
#pragma unroll
      for (int w = 0; w < kPartWarps; ++w) {
#pragma unroll
        for (int i = 0; i < kO; ++i) {
          const uint32_t a = sm.wcnt[w][lane + 32 * i];
          sm.wcnt[w][lane + 32 * i] = t[i];
          t[i] += a;
        }
      }
      uint32_t sc[kO];
#pragma unroll
      for (int i = 0; i < kO; ++i) sc[i] = t[i];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int i = 0; i < kO; ++i) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, sc[i], d);
          if (lane >= static_cast<uint32_t>(d)) sc[i] += y;
        }
      }
      uint16_t* bo = boffs + ch * kBoffStride;
      // buckets >= S are empty: their offsets equal cnt (lanes >= S may hold
      // counts of aliased ids, which no key uses)
      uint32_t carry = 0;
#pragma unroll
      for (int i = 0; i < kChunkBuckets / 32; ++i) {
        const uint32_t b = lane + 32 * i;
        uint32_t o = cnt;
        if (i < kO) {
          o = carry + sc[i] - t[i];
          carry += __shfl_sync(0xffffffffu, sc[i], 31);
          sm.boff[b] = o;
        }
        bo[b] = static_cast<uint16_t>(b < bm.S ? o : cnt);
      }
      if (lane == 0) bo[kChunkBuckets] = static_cast<uint16_t>(cnt);
    }
    __syncthreads();
    uint32_t sbase[owned<BITS>()];
#pragma unroll
    for (int i = 0; i < owned<BITS>(); ++i) sbase[i] = sm.boff[lane + 32 * i] + sm.wcnt[warp][lane + 32 * i];
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint32_t loc = slot_base<BITS>(bk[j], sbase) + off[j];
      if (bk[j] != 0xffffffffu) {
        SBBF_DCHECK(loc < cnt && bk[j] < bm.S && loc == sm.boff[bk[j]] + sm.wcnt[warp][bk[j]] + off[j]);
        sm.key[loc] = slot_value<kTop>(h[j], bk[j], j * kPartThreads + threadIdx.x, bm, starts);
        if (!bm.pack) sm.pos[loc] = static_cast<uint16_t>(j * kPartThreads + threadIdx.x);
      }
    }
    __syncthreads();
    if (cnt == kPartChunk) {
      // 16-byte copies: two keys / eight positions per thread per step
      const uint4* ks = reinterpret_cast<const uint4*>(sm.key);
      uint4* ko = reinterpret_cast<uint4*>(out + base);
      for (uint32_t v = threadIdx.x; v < kPartChunk / 2; v += kPartThreads) ko[v] = ks[v];
      if (pos16) {
        const uint4* ps = reinterpret_cast<const uint4*>(sm.pos);
        uint4* po = reinterpret_cast<uint4*>(pos16 + base);
        for (uint32_t v = threadIdx.x; v < kPartChunk / 8; v += kPartThreads) po[v] = ps[v];
      }
    } else {
      for (uint32_t i = threadIdx.x; i < cnt; i += kPartThreads) {
        out[base + i] = sm.key[i];
        if (pos16) pos16[base + i] = sm.pos[i];
      }
    }
    __syncthreads();
  }
}

// chunk_scatter with the data movement on the TMA engine: each CTA's next
// chunk of keys is bulk-loaded (cp.async.bulk + mbarrier) into a second
// input buffer while this one is ranked, and the bucket-major staging is
// written out by bulk stores (cp.async.bulk.global.shared::cta), so the
// threads only read keys from shared memory, rank and place them. Full
// chunks with 16-byte aligned keys only; the caller sends a partial last
// chunk through chunk_scatter_kernel.
struct ChunkTmaSmem {
  uint64_t in[2][kPartChunk];  // input ring (bulk loads)
  uint64_t key[kPartChunk];    // bucket-major staging (bulk stores)
  alignas(16) uint16_t pos[kPartChunk];
  uint32_t wcnt[kPartWarps][kChunkBuckets];
  uint32_t boff[kChunkBuckets + 1];
  alignas(8) uint64_t bar[2];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_addr(bar)), "r"(parity)
                 : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}

template <int BITS, bool kTop>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks)
    chunk_scatter_tma_kernel(const uint64_t* __restrict__ hashes, uint64_t nfull, BucketMap bm,
                             uint64_t* __restrict__ out, uint16_t* __restrict__ pos16, uint16_t* __restrict__ boffs) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ChunkTmaSmem& sm = *reinterpret_cast<ChunkTmaSmem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OwnerMasks om(lane);
  constexpr uint32_t kBytes = kPartChunk * sizeof(uint64_t);
  // packed maps write no positions: the array's space holds the bucket starts
  uint64_t* const starts = reinterpret_cast<uint64_t*>(sm.pos);
  fill_starts<kTop>(bm, starts);
  if (bm.pack) pos16 = nullptr;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    if (blockIdx.x < nfull) bulk_load(sm.in[0], hashes + blockIdx.x * kPartChunk, kBytes, &sm.bar[0]);
  }
  __syncthreads();
  uint32_t it = 0;
  for (uint64_t ch = blockIdx.x; ch < nfull; ch += gridDim.x, ++it) {
    const uint32_t k = it & 1;
    const uint64_t base = ch * kPartChunk;
    if (threadIdx.x == 0 && ch + gridDim.x < nfull) {
      // the other buffer's last readers passed this iteration's barriers
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(sm.in[k ^ 1], hashes + (ch + gridDim.x) * kPartChunk, kBytes, &sm.bar[k ^ 1]);
    }
    bulk_wait(&sm.bar[k], (it >> 1) & 1);
    uint64_t h[kPartPerThread];
    uint32_t bk[kPartPerThread], off[kPartPerThread];
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) h[j] = sm.in[k][j * kPartThreads + threadIdx.x];
    uint32_t c[owned<BITS>()] = {};
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      bk[j] = bucket_of<kTop>(h[j], bm);
      off[j] = warp_rank<BITS>(bk[j], true, lane, om, c);
    }
#pragma unroll
    for (int i = 0; i < kChunkBuckets / 32; ++i) sm.wcnt[warp][lane + 32 * i] = i < owned<BITS>() ? c[i] : 0u;
    __syncthreads();
    if (warp == 0) {
      constexpr int kO = owned<BITS>();
      uint32_t t[kO] = {};
#pragma unroll
      for (int w = 0; w < kPartWarps; ++w) {
#pragma unroll
        for (int i = 0; i < kO; ++i) {
          const uint32_t a = sm.wcnt[w][lane + 32 * i];
          sm.wcnt[w][lane + 32 * i] = t[i];
          t[i] += a;
        }
      }
      uint32_t sc[kO];
#pragma unroll
      for (int i = 0; i < kO; ++i) sc[i] = t[i];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int i = 0; i < kO; ++i) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, sc[i], d);
          if (lane >= static_cast<uint32_t>(d)) sc[i] += y;
        }
      }
      uint16_t* bo = boffs + ch * kBoffStride;
      uint32_t carry = 0;
#pragma unroll
      for (int i = 0; i < kChunkBuckets / 32; ++i) {
        const uint32_t b = lane + 32 * i;
        uint32_t o = kPartChunk;
        if (i < kO) {
          o = carry + sc[i] - t[i];
          carry += __shfl_sync(0xffffffffu, sc[i], 31);
          sm.boff[b] = o;
        }
        bo[b] = static_cast<uint16_t>(b < bm.S ? o : kPartChunk);
      }
      if (lane == 0) {
        bo[kChunkBuckets] = static_cast<uint16_t>(kPartChunk);
        // the previous chunk's bulk stores have finished reading the staging
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    __syncthreads();
    uint32_t sbase[owned<BITS>()];
#pragma unroll
    for (int i = 0; i < owned<BITS>(); ++i) sbase[i] = sm.boff[lane + 32 * i] + sm.wcnt[warp][lane + 32 * i];
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint32_t loc = slot_base<BITS>(bk[j], sbase) + off[j];
      SBBF_DCHECK(loc < kPartChunk && bk[j] < bm.S);
      sm.key[loc] = slot_value<kTop>(h[j], bk[j], j * kPartThreads + threadIdx.x, bm, starts);
      if (!bm.pack) sm.pos[loc] = static_cast<uint16_t>(j * kPartThreads + threadIdx.x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_store(out + base, sm.key, kBytes);
      if (pos16) bulk_store(pos16 + base, sm.pos, kPartChunk * sizeof(uint16_t));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Probe (lookup) or OR (insert) bucket by bucket: CTA blockIdx handles bucket
// b = blockIdx / groups over chunks [grp*G, grp*G + G); CTAs run in blockIdx
// order, so the keys in flight all fall in one or two ~32 MiB filter slices
// and their sectors / atomics are served by L2. Each warp works on 4 chunk
// segments at a time (independent loads in flight); a segment is the
// chunk's contiguous run of bucket b. Lookups store one answer byte per
// routed slot (plain stores, no atomics).
constexpr int kSegThreads = 256;
constexpr int kSegWarps = kSegThreads / 32;
constexpr uint32_t kSegChunksPerCta = 64;
// chunks per work item of the persistent segment grid (SBBF_SEG_ITEM_CHUNKS: A/B only)
uint32_t seg_items_chunks() {
  static const uint32_t v = [] {
    const char* e = getenv("SBBF_SEG_ITEM_CHUNKS");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? static_cast<uint32_t>(x) : 16u;
  }();
  return v;
}
// SBBF_SEG_CHUNKS overrides the chunks per segment CTA (A/B only)
// Config 4 (profiles/r2_ab/r2au_*, r2ax_*): inserts 16 chunks per CTA at 2
// segments per warp step, lookups 64 (107.1 vs 105.4 at 32; 96: 101.3, 128: 90.3).
uint32_t seg_chunks_per_cta(bool insert) {
  static const uint32_t v = [] {
    const char* e = getenv("SBBF_SEG_CHUNKS");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? static_cast<uint32_t>(x) : 0u;
  }();
  return v ? v : insert ? kSegChunksPerCta / 4 : kSegChunksPerCta;
}

// One work item: bucket b over chunks [c_begin, c_end).
// Insert dedup table (kDedup): a per-CTA direct-mapped set of the hashes this
// CTA has already ORed, indexed by the hash's low bits. Entry e starts as
// e ^ 1, which no hash indexed to e can equal, so a hit is always a hash this
// CTA has issued its reds for and skipping it is exact (OR is idempotent and
// the reds land before the kernel ends). It replaces the test-before-set load:
// config 4's hot keys are caught in shared memory, and distinct keys cost one
// L2 atomic instead of a test load plus an atomic.
constexpr uint32_t kDedupSlots = 2048;

template <bool kInsert, int kSegQ, bool kDedup = false>
__device__ __forceinline__ void segment_item(uint32_t* __restrict__ blocks, const Geom& g,
                                             const uint64_t* __restrict__ keys, const uint16_t* __restrict__ boffs,
                                             uint64_t m, uint8_t* __restrict__ ans, uint32_t b, uint64_t c_begin,
                                             uint64_t c_end, uint64_t* __restrict__ dtab = nullptr) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t keep = dev::policy_evict_last();
  for (uint64_t c = c_begin + warp * kSegQ; c < c_end; c += kSegWarps * kSegQ) {
    uint64_t seg[kSegQ];
    uint32_t len[kSegQ];
    uint32_t maxlen = 0;
#pragma unroll
    for (int q = 0; q < kSegQ; ++q) {
      const uint64_t ch = c + q;
      uint32_t st = 0, en = 0;
      if (ch < c_end) {
        st = boffs[ch * kBoffStride + b];
        en = boffs[ch * kBoffStride + b + 1];
        SBBF_DCHECK(st <= en && en <= boffs[ch * kBoffStride + kChunkBuckets] && ch * kPartChunk + en <= m);
      }
      seg[q] = ch * kPartChunk + st;
      len[q] = en - st;
      maxlen = len[q] > maxlen ? len[q] : maxlen;
    }
    if constexpr (kInsert) {
      // 4 lanes per key, one 64-bit lane pair each (as insert_wide_kernel);
      // test-before-set: grouped duplicates (config 4's hot keys) skip the
      // atomic, and their test loads hit L1 (.ca: .cg / .nc measured slower)
      const uint32_t pair = lane & 3;
      const uint32_t seed_lo = dev::lane_seed_rt(2 * pair), seed_hi = dev::lane_seed_rt(2 * pair + 1);
      uint64_t hn[kSegQ];
#pragma unroll
      for (int q = 0; q < kSegQ; ++q)
        hn[q] = (lane >> 2) < len[q] ? dev::ld_stream_u64(keys + seg[q] + (lane >> 2), pol) : 0;
      // warp-uniform trip count (the dedup path synchronises the warp)
      for (uint32_t j0 = 0; j0 < maxlen; j0 += 8) {
        const uint32_t j = j0 + (lane >> 2);
        uint64_t h[kSegQ];
#pragma unroll
        for (int q = 0; q < kSegQ; ++q) h[q] = hn[q];
        uint64_t* ptr[kSegQ];
        uint64_t mask[kSegQ], cur[kSegQ];
#pragma unroll
        for (int q = 0; q < kSegQ; ++q) {
          const uint64_t blk = dev::block_index(h[q], g.nb_global) - g.first;
          const bool ok = j < len[q] && blk < g.nb_local;
          const uint32_t low = static_cast<uint32_t>(h[q]);
          ptr[q] = reinterpret_cast<uint64_t*>(blocks + (ok ? blk : 0) * 8) + pair;
          mask[q] = ok ? (static_cast<uint64_t>(dev::lane_bit(low, seed_hi)) << 32) | dev::lane_bit(low, seed_lo) : 0;
          if constexpr (kDedup) {
            cur[q] = mask[q] && dtab[low & (kDedupSlots - 1)] == h[q] ? ~0ull : 0;
          } else {
            cur[q] = mask[q] ? dev::ld_pair(ptr[q], keep) : ~0ull;
          }
        }
        if constexpr (kDedup) {
          // every lane of a key has read the table before any records it
          __syncwarp();
#pragma unroll
          for (int q = 0; q < kSegQ; ++q)
            if (pair == 0 && mask[q] && !cur[q]) dtab[static_cast<uint32_t>(h[q]) & (kDedupSlots - 1)] = h[q];
        }
#pragma unroll
        for (int q = 0; q < kSegQ; ++q) hn[q] = j + 8 < len[q] ? dev::ld_stream_u64(keys + seg[q] + j + 8, pol) : 0;
#pragma unroll
        for (int q = 0; q < kSegQ; ++q)
          if (mask[q] & ~cur[q]) dev::red_or64(ptr[q], mask[q], keep);
      }
    } else {
      // the next step's keys load while this step's sectors are in flight
      uint64_t hn[kSegQ];
#pragma unroll
      for (int q = 0; q < kSegQ; ++q) hn[q] = lane < len[q] ? dev::ld_stream_u64(keys + seg[q] + lane, pol) : 0;
      for (uint32_t j = lane; j < maxlen; j += 32) {
        uint64_t h[kSegQ];
#pragma unroll
        for (int q = 0; q < kSegQ; ++q) h[q] = hn[q];
        dev::Block8 bl[kSegQ];
        uint32_t owned = 0;
#pragma unroll
        for (int q = 0; q < kSegQ; ++q) {
          const uint64_t blk = dev::block_index(h[q], g.nb_global) - g.first;
          const bool ok = blk < g.nb_local;
          owned |= static_cast<uint32_t>(ok) << q;
          dev::ld_block_nc_normal(blocks + (ok ? blk : 0) * 8, bl[q]);
        }
#pragma unroll
        for (int q = 0; q < kSegQ; ++q)
          hn[q] = j + 32 < len[q] ? dev::ld_stream_u64(keys + seg[q] + j + 32, pol) : 0;
#pragma unroll
        for (int q = 0; q < kSegQ; ++q)
          if (j < len[q]) ans[seg[q] + j] = (((owned >> q) & 1u) && dev::block_contains(bl[q], h[q])) ? 1 : 0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// tile insert (filters beyond L2, whole power-of-two filters)
// ---------------------------------------------------------------------------
// The segment sweep ORs keys into an L2-resident slice with one L2 atomic
// (plus a test load) per key, ~55-65 G/s whatever the MLP (profiles/r2_ab).
// The tile path instead applies each 64 KiB tile of the filter in shared
// memory: a second partition groups every slice's keys by tile, then one CTA
// per tile bulk-loads the tile, ORs its keys with shared-memory atomics and
// bulk-stores it back, so the filter streams through HBM once per call and
// no key touches L2 atomically.
//   1. chunk_scatter(_tma): keys chunk-local by slice (S = nb / 2^19 slices
//      of 256 tiles), as the other paths;
//   2. tile_scatter_kernel: CTA (slice b, chunk group g) gathers its chunks'
//      runs of slice b and writes them tile-major into the same positions of
//      a second buffer (group g's region, slice b's share of it), with the
//      absolute start of every tile's run (tile_runs[b][g][0..256]);
//   3. tile_apply_persistent_kernel: persistent CTAs apply tile t's G runs
//      in shared memory, tile after tile.
constexpr int kTileBits = 8;
constexpr uint32_t kTilesPerSlice = 1u << kTileBits;
constexpr uint32_t kTileBlocks = 2048;  // 64 KiB
constexpr int kTileLog2 = 11;
constexpr uint32_t kTileGroupChunks = 48;  // chunks per tile_scatter CTA (~3072 keys: one smem piece)
constexpr uint32_t kTileSegTable = 64;     // run-table capacity (warp-0 scan: 2 entries per lane)
constexpr int kTileScatterThreads = 512;
constexpr int kTileScatterWarps = kTileScatterThreads / 32;
constexpr int kTilePiece = 4096;           // keys placed per smem pass
constexpr int kTilePerThread = kTilePiece / kTileScatterThreads;

struct TileScatterSmem {
  uint64_t key[kTilePiece];   // one piece staged tile-major
  uint8_t tile[kTilePiece];
  uint16_t kp[kTilePiece + 1];  // exclusive prefix of kept slots (staged order); kp[pn] = kept
  union {
    uint32_t wcnt[kTileScatterWarps][kTilesPerSlice];  // multisplit counters (several pieces)
    uint32_t map[kTilePiece];                          // flat position -> key index (one piece)
  } u;
  uint32_t poff[kTilesPerSlice];  // piece-local staged offset of each tile (before dedup)
  uint32_t off[kTilesPerSlice];   // CTA: kept-key offset of each tile (several pieces)
  uint32_t cur[kTilesPerSlice];   // CTA: kept keys of each tile written so far
  uint32_t wsum[kTileScatterWarps];
  uint32_t s_start[kTileSegTable];
  uint32_t s_pre[kTileSegTable + 1];
  uint32_t s_st[kTileSegTable];
};

// key index of flat position pos within the CTA's runs: the last run whose
// prefix is <= pos, by binary search over s_pre[0..nseg) (empty runs share
// their successor's prefix, so the last match is the non-empty one). seg is
// kept for the callers' interface: a lower bound that only advances.
__device__ __forceinline__ uint32_t flat_key(const uint32_t* s_start, const uint32_t* s_pre, uint32_t nseg,
                                             uint32_t pos, uint32_t& seg) {
  uint32_t lo = seg, hi = nseg;  // invariant: s_pre[lo] <= pos, answer in [lo, hi)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s_pre[mid] <= pos) lo = mid;
    else hi = mid;
  }
  seg = lo;
  return s_start[lo] + (pos - s_pre[lo]);
}

// Warp 0: per-tile totals over the warps' counters (wcnt becomes each warp's
// exclusive prefix per tile) and their exclusive prefix over tiles (out).
__device__ __forceinline__ void tile_scan_warp0(uint32_t (&wcnt)[kTileScatterWarps][kTilesPerSlice], uint32_t* out,
                                                uint32_t lane) {
  constexpr int kO = kTilesPerSlice / 32;
  uint32_t t[kO] = {};
#pragma unroll
  for (int w = 0; w < kTileScatterWarps; ++w) {
#pragma unroll
    for (int i = 0; i < kO; ++i) {
      const uint32_t a = wcnt[w][lane + 32 * i];
      wcnt[w][lane + 32 * i] = t[i];
      t[i] += a;
    }
  }
  uint32_t sc[kO];
#pragma unroll
  for (int i = 0; i < kO; ++i) sc[i] = t[i];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int i = 0; i < kO; ++i) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, sc[i], d);
      if (lane >= static_cast<uint32_t>(d)) sc[i] += y;
    }
  }
  uint32_t carry = 0;
#pragma unroll
  for (int i = 0; i < kO; ++i) {
    out[lane + 32 * i] = carry + sc[i] - t[i];
    carry += __shfl_sync(0xffffffffu, sc[i], 31);
  }
}

// Exclusive prefix of a[0..256) over tiles into out (warp 0; a and out may alias).
__device__ __forceinline__ uint32_t scan256_warp0(const uint32_t* a, uint32_t* out, uint32_t lane) {
  constexpr int kO = kTilesPerSlice / 32;
  uint32_t v[kO], run = 0;
#pragma unroll
  for (int i = 0; i < kO; ++i) {
    v[i] = a[lane * kO + i];
    run += v[i];
  }
  __syncwarp();
  uint32_t incl = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= static_cast<uint32_t>(d)) incl += y;
  }
  uint32_t acc = incl - run;
#pragma unroll
  for (int i = 0; i < kO; ++i) {
    out[lane * kO + i] = acc;
    acc += v[i];
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

__device__ __forceinline__ void tile_dedup(TileScatterSmem& sm, uint32_t pn, uint32_t lane, uint32_t warp);

// One piece of up to kTilePiece flat keys: loaded, ranked by tile, staged
// tile-major in smem, then de-duplicated — a slot whose key equals the slot
// before it in the same tile's run is dropped (config 4's hot keys arrive as
// long runs of one key: ~99 % of a hot tile's slots). On return (after a
// barrier): sm.key/tile staged, sm.poff the staged tile offsets, sm.kp the
// kept-slot prefix (kp[pn] = kept keys).
__device__ __forceinline__ void tile_piece(TileScatterSmem& sm, const uint64_t* __restrict__ keys, uint32_t p0,
                                           uint32_t pn, uint32_t nseg, uint32_t& seg, uint64_t nb, uint64_t slice_first,
                                           uint64_t pol, const OwnerMasks& om, uint32_t lane, uint32_t warp) {
  uint64_t h[kTilePerThread];
  uint32_t tl[kTilePerThread], off[kTilePerThread];
  uint32_t c[owned<kTileBits>()] = {};
#pragma unroll
  for (int j = 0; j < kTilePerThread; ++j) {
    const uint32_t i = j * kTileScatterThreads + threadIdx.x;
    h[j] = i < pn ? dev::ld_stream_u64(keys + flat_key(sm.s_start, sm.s_pre, nseg, p0 + i, seg), pol) : 0;
  }
#pragma unroll
  for (int j = 0; j < kTilePerThread; ++j) {
    const uint32_t i = j * kTileScatterThreads + threadIdx.x;
    const bool valid = i < pn;
    tl[j] = valid ? static_cast<uint32_t>((dev::block_index(h[j], nb) - slice_first) >> kTileLog2) : 0;
    off[j] = warp_rank<kTileBits>(tl[j], valid, lane, om, c);
    if (!valid) tl[j] = 0xffffffffu;
  }
#pragma unroll
  for (int i = 0; i < owned<kTileBits>(); ++i) sm.u.wcnt[warp][lane + 32 * i] = c[i];
  __syncthreads();
  if (warp == 0) tile_scan_warp0(sm.u.wcnt, sm.poff, lane);
  __syncthreads();
  uint32_t sbase[owned<kTileBits>()];
#pragma unroll
  for (int i = 0; i < owned<kTileBits>(); ++i) sbase[i] = sm.poff[lane + 32 * i] + sm.u.wcnt[warp][lane + 32 * i];
#pragma unroll
  for (int j = 0; j < kTilePerThread; ++j) {
    const uint32_t loc = slot_base<kTileBits>(tl[j] & 0xffu, sbase) + off[j];
    if (tl[j] != 0xffffffffu) {
      SBBF_DCHECK(loc < pn);
      sm.key[loc] = h[j];
      sm.tile[loc] = static_cast<uint8_t>(tl[j]);
    }
  }
  __syncthreads();
  tile_dedup(sm, pn, lane, warp);
}

// Drop staged slots whose key equals the previous slot of the same tile run;
// sm.kp = exclusive prefix of the kept slots (kp[pn] = kept). Ends on a barrier.
__device__ __forceinline__ void tile_dedup(TileScatterSmem& sm, uint32_t pn, uint32_t lane, uint32_t warp) {
  // keep flags of 8 consecutive staged slots per thread, block-wide prefix
  const uint32_t i0 = threadIdx.x * kTilePerThread;
  uint32_t keep = 0, cnt = 0;
#pragma unroll
  for (int k = 0; k < kTilePerThread; ++k) {
    const uint32_t i = i0 + k;
    bool kept = false;
    if (i < pn) {
      const uint32_t t = sm.tile[i];
      kept = !(i > sm.poff[t] && sm.key[i] == sm.key[i - 1]);
    }
    keep |= static_cast<uint32_t>(kept) << k;
    cnt += kept;
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= static_cast<uint32_t>(d)) incl += y;
  }
  if (lane == 31) sm.wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < kTileScatterWarps ? sm.wsum[lane] : 0;
    uint32_t wi = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= static_cast<uint32_t>(d)) wi += y;
    }
    if (lane < kTileScatterWarps) sm.wsum[lane] = wi - v;
  }
  __syncthreads();
  uint32_t run = sm.wsum[warp] + incl - cnt;
#pragma unroll
  for (int k = 0; k < kTilePerThread; ++k) {
    const uint32_t i = i0 + k;
    if (i <= pn) sm.kp[i] = static_cast<uint16_t>(run);
    run += (keep >> k) & 1u;
  }
  if (i0 + kTilePerThread == pn) sm.kp[pn] = static_cast<uint16_t>(run);
  __syncthreads();
}

__global__ void __launch_bounds__(kTileScatterThreads, 2)
    tile_scatter_kernel(uint64_t nb, uint32_t S, const uint64_t* __restrict__ keys, const uint16_t* __restrict__ boffs,
                        uint64_t m, uint32_t groups, uint64_t* __restrict__ out, uint32_t* __restrict__ runs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileScatterSmem& sm = *reinterpret_cast<TileScatterSmem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OwnerMasks om(lane);
  const uint32_t b = blockIdx.x / groups, g = blockIdx.x % groups;
  const uint64_t nchunks = (m + kPartChunk - 1) / kPartChunk;
  const uint64_t c0 = static_cast<uint64_t>(g) * kTileGroupChunks;
  const uint32_t nseg = static_cast<uint32_t>(c0 + kTileGroupChunks < nchunks ? kTileGroupChunks : nchunks - c0);
  const uint64_t slice_first = static_cast<uint64_t>(b) * (nb / S);
  const uint64_t pol = dev::policy_evict_first();
  // segment table: run starts, prefix of lengths; this CTA's output base =
  // group region + the keys of slices < b in the group's chunks
  if (threadIdx.x < kTileSegTable) {
    uint32_t st = 0, len = 0;
    if (threadIdx.x < nseg) {
      const uint64_t ch = c0 + threadIdx.x;
      st = boffs[ch * kBoffStride + b];
      len = boffs[ch * kBoffStride + b + 1] - st;
      sm.s_start[threadIdx.x] = static_cast<uint32_t>(ch * kPartChunk + st);
    }
    sm.s_st[threadIdx.x] = st;
    sm.s_pre[threadIdx.x + 1] = len;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t v0 = sm.s_pre[1 + 2 * lane], v1 = sm.s_pre[2 + 2 * lane];
    uint32_t a0 = sm.s_st[2 * lane] + sm.s_st[2 * lane + 1];
    __syncwarp();
    uint32_t incl = v0 + v1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= static_cast<uint32_t>(d)) incl += y;
    }
    sm.s_pre[2 * lane] = incl - v0 - v1;
    sm.s_pre[2 * lane + 1] = incl - v1;
    if (lane == 31) sm.s_pre[kTileSegTable] = incl;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, d);
    if (lane == 0) sm.s_st[0] = a0;  // sum of starts: keys of slices < b in the group
  }
  __syncthreads();
  const uint32_t n = sm.s_pre[nseg];
  const uint64_t base = c0 * kPartChunk + sm.s_st[0];
  uint32_t* r = runs + static_cast<uint64_t>(blockIdx.x) * (kTilesPerSlice + 1);
  if (n <= static_cast<uint32_t>(kTilePiece)) {
    // One piece: a counting sort by tile through shared-memory atomics (tile
    // order within a run does not matter for inserts), keys addressed through
    // a flat-position map built from the run table. Staged order is the
    // output order (kept slots only).
    for (uint32_t r = warp; r < nseg; r += kTileScatterWarps) {
      const uint32_t st = sm.s_start[r], p = sm.s_pre[r], len = sm.s_pre[r + 1] - p;
      for (uint32_t k = lane; k < len; k += 32) sm.u.map[p + k] = st + k;
    }
    for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads) sm.off[t] = 0;
    __syncthreads();
    uint64_t h[kTilePerThread];
    uint32_t tl[kTilePerThread];
#pragma unroll
    for (int j = 0; j < kTilePerThread; ++j) {
      const uint32_t f = j * kTileScatterThreads + threadIdx.x;
      h[j] = f < n ? dev::ld_stream_u64(keys + sm.u.map[f], pol) : 0;
    }
#pragma unroll
    for (int j = 0; j < kTilePerThread; ++j) {
      const uint32_t f = j * kTileScatterThreads + threadIdx.x;
      tl[j] = static_cast<uint32_t>((dev::block_index(h[j], nb) - slice_first) >> kTileLog2);
      if (f < n) atomicAdd(&sm.off[tl[j]], 1u);
    }
    __syncthreads();
    if (warp == 0) scan256_warp0(sm.off, sm.poff, lane);
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads) sm.cur[t] = sm.poff[t];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTilePerThread; ++j) {
      if (j * kTileScatterThreads + threadIdx.x < n) {
        const uint32_t pos = atomicAdd(&sm.cur[tl[j]], 1u);
        sm.key[pos] = h[j];
        sm.tile[pos] = static_cast<uint8_t>(tl[j]);
      }
    }
    __syncthreads();
    tile_dedup(sm, n, lane, warp);
    for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads)
      r[t] = static_cast<uint32_t>(base + sm.kp[sm.poff[t]]);
    if (threadIdx.x == 0) r[kTilesPerSlice] = static_cast<uint32_t>(base + sm.kp[n]);
    for (uint32_t i = threadIdx.x; i < n; i += kTileScatterThreads)
      if (sm.kp[i + 1] != sm.kp[i]) out[base + sm.kp[i]] = sm.key[i];
    return;
  }
  // several pieces: pass 1 counts the kept keys per tile, pass 2 writes them
  for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads) sm.off[t] = 0;
  uint32_t seg = 0;
  for (uint32_t p0 = 0; p0 < n; p0 += kTilePiece) {
    const uint32_t pn = n - p0 < static_cast<uint32_t>(kTilePiece) ? n - p0 : kTilePiece;
    tile_piece(sm, keys, p0, pn, nseg, seg, nb, slice_first, pol, om, lane, warp);
    for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads) {
      const uint32_t e = t + 1 < kTilesPerSlice ? sm.poff[t + 1] : pn;
      sm.off[t] += sm.kp[e] - sm.kp[sm.poff[t]];
    }
    __syncthreads();
  }
  if (warp == 0) {
    const uint32_t total = scan256_warp0(sm.off, sm.off, lane);
    if (lane == 0) r[kTilesPerSlice] = static_cast<uint32_t>(base + total);
  }
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads) {
    r[t] = static_cast<uint32_t>(base + sm.off[t]);
    sm.cur[t] = 0;
  }
  __syncthreads();
  seg = 0;
  for (uint32_t p0 = 0; p0 < n; p0 += kTilePiece) {
    const uint32_t pn = n - p0 < static_cast<uint32_t>(kTilePiece) ? n - p0 : kTilePiece;
    tile_piece(sm, keys, p0, pn, nseg, seg, nb, slice_first, pol, om, lane, warp);
    for (uint32_t i = threadIdx.x; i < pn; i += kTileScatterThreads)
      if (sm.kp[i + 1] != sm.kp[i]) {
        const uint32_t t = sm.tile[i];
        const uint64_t dst = base + sm.off[t] + sm.cur[t] + (sm.kp[i] - sm.kp[sm.poff[t]]);
        SBBF_DCHECK(dst < m);
        out[dst] = sm.key[i];
      }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < kTilesPerSlice; t += kTileScatterThreads) {
      const uint32_t e = t + 1 < kTilesPerSlice ? sm.poff[t + 1] : pn;
      sm.cur[t] += sm.kp[e] - sm.kp[sm.poff[t]];
    }
    __syncthreads();
  }
}

constexpr uint32_t kTileMaxGroups = 1024;  // runs per tile held in smem (host check)

// Persistent tile apply: one CTA per SM walks its tiles (c, c + grid, ...)
// in sweep order with three 64 KiB tile buffers — the tile two ahead loads by
// TMA while this one is applied and the previous one is stored — and the next
// tile's run table prefetched. One thread per key (all of a tile's keys in
// flight at once for tiles up to 4 keys per thread); each thread walks its
// block's eight words from a rotated start so a warp's shared accesses spread
// over the banks.
constexpr int kTileP2Threads = 1024;
constexpr int kTileP2Bufs = 3;
constexpr int kTileP2U = 4;

struct TileApply2Smem {
  uint32_t w[kTileP2Bufs][kTileBlocks * 8];
  uint32_t r_lo[2][kTileMaxGroups];
  uint32_t r_pre[2][kTileMaxGroups + 1];
  uint32_t seeds[8];
  alignas(8) uint64_t bar[kTileP2Bufs];
};

__global__ void __launch_bounds__(kTileP2Threads, 1)
    tile_apply_persistent_kernel(uint32_t* __restrict__ blocks, uint64_t nb, uint32_t S,
                                 const uint64_t* __restrict__ keys, const uint32_t* __restrict__ runs, uint32_t groups,
                                 uint32_t rev) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileApply2Smem& sm = *reinterpret_cast<TileApply2Smem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ntiles = S * kTilesPerSlice;
  const uint64_t slice_blocks = nb / S;
  constexpr uint32_t kBytes = kTileBlocks * 32;
  auto tile_of = [&](uint32_t k) -> uint32_t { return rev ? ntiles - 1 - k : k; };  // k-th tile of the sweep
  auto first_block = [&](uint32_t bt) -> uint64_t {
    return static_cast<uint64_t>(bt >> kTileBits) * slice_blocks + static_cast<uint64_t>(bt & (kTilesPerSlice - 1)) * kTileBlocks;
  };
  auto issue_load = [&](uint32_t k, uint32_t buf) {
    const uint32_t* src = blocks + first_block(tile_of(k)) * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&sm.bar[buf])), "r"(kBytes)
                 : "memory");
#pragma unroll
    for (uint32_t o = 0; o < kBytes; o += 16384)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(reinterpret_cast<char*>(sm.w[buf]) + o)),
                   "l"(reinterpret_cast<const char*>(src) + o), "r"(16384u), "r"(smem_addr(&sm.bar[buf]))
                   : "memory");
  };
  auto load_runs = [&](uint32_t k, uint32_t rb) {
    const uint32_t bt = tile_of(k), b = bt >> kTileBits, t = bt & (kTilesPerSlice - 1);
    for (uint32_t g = threadIdx.x; g < groups; g += kTileP2Threads) {
      const uint32_t* r = runs + (static_cast<uint64_t>(b) * groups + g) * (kTilesPerSlice + 1) + t;
      const uint32_t lo = r[0], hi = r[1];
      sm.r_lo[rb][g] = lo;
      sm.r_pre[rb][g + 1] = hi - lo;
    }
  };
  if (threadIdx.x < 8) sm.seeds[threadIdx.x] = dev::lane_seed_rt(static_cast<int>(threadIdx.x));
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kTileP2Bufs; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    if (blockIdx.x < ntiles) issue_load(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < ntiles) issue_load(blockIdx.x + gridDim.x, 1);
  }
  if (blockIdx.x < ntiles) load_runs(blockIdx.x, 0);
  const uint64_t pol = dev::policy_evict_first();
  uint32_t it = 0;
  for (uint32_t k = blockIdx.x; k < ntiles; k += gridDim.x, ++it) {
    const uint32_t buf = it % kTileP2Bufs, rb = it & 1;
    __syncthreads();  // run table rb written; previous tile's apply done
    if (warp == 0) {
      uint32_t carry = 0;
      for (uint32_t g0 = 0; g0 < groups; g0 += 32) {
        const uint32_t g = g0 + lane;
        const uint32_t v = g < groups ? sm.r_pre[rb][g + 1] : 0;
        uint32_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= static_cast<uint32_t>(d)) incl += y;
        }
        __syncwarp();
        if (g < groups) sm.r_pre[rb][g] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) sm.r_pre[rb][groups] = carry;
    }
    __syncthreads();
    // the next tile's run table loads while this one is applied
    if (k + gridDim.x < ntiles) load_runs(k + gridDim.x, rb ^ 1);
    const uint32_t n = sm.r_pre[rb][groups];
    const uint64_t tfirst = first_block(tile_of(k));
    uint32_t seg = 0;
    // keys of this thread: f = base + u * 1024 + tid
    uint64_t h[kTileP2U];
#pragma unroll
    for (int u = 0; u < kTileP2U; ++u) {
      const uint32_t f = u * kTileP2Threads + threadIdx.x;
      h[u] = f < n ? dev::ld_stream_u64(keys + flat_key(sm.r_lo[rb], sm.r_pre[rb], groups, f, seg), pol) : 0;
    }
    bulk_wait(&sm.bar[buf], (it / kTileP2Bufs) & 1);
    uint32_t* tw = sm.w[buf];
    for (uint32_t base = 0; base < n; base += kTileP2U * kTileP2Threads) {
#pragma unroll
      for (int u = 0; u < kTileP2U; ++u) {
        const uint32_t f = base + u * kTileP2Threads + threadIdx.x;
        if (f < n) {
          const uint32_t blk = static_cast<uint32_t>(dev::block_index(h[u], nb) - tfirst);
          SBBF_DCHECK(blk < kTileBlocks);
          const uint32_t low = static_cast<uint32_t>(h[u]);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t wi = (i + threadIdx.x) & 7;
            const uint32_t bit = dev::lane_bit(low, sm.seeds[wi]);
            uint32_t* p = tw + blk * 8 + wi;
            if ((*p & bit) == 0) atomicOr(p, bit);
          }
        }
      }
      const uint32_t nb2 = base + kTileP2U * kTileP2Threads;
      if (nb2 < n) {
#pragma unroll
        for (int u = 0; u < kTileP2U; ++u) {
          const uint32_t f = nb2 + u * kTileP2Threads + threadIdx.x;
          h[u] = f < n ? dev::ld_stream_u64(keys + flat_key(sm.r_lo[rb], sm.r_pre[rb], groups, f, seg), pol) : 0;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_store(blocks + tfirst * 8, tw, kBytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the tile two ahead goes into the buffer whose store was committed last
      // iteration: wait until that store has read it
      const uint32_t k2 = k + 2 * gridDim.x;
      if (k2 < ntiles) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_load(k2, (it + 2) % kTileP2Bufs);
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Items are (bucket, group of per_cta chunks) in bucket-major order. With
// `work` null the grid has one CTA per item (blockIdx order); otherwise the
// grid is the resident CTAs and each takes the next item from a global
// counter, so the items in flight — and the filter slices live in L2 — stay
// within about one resident wave of small items whatever the CTA duration
// spread (a one-shot grid of 64-chunk items keeps 2-3 slices live and reads
// each slice ~3x from HBM: profiles/r2_*).
template <bool kInsert, int kSegQ, int kMinB = (kSegQ > 4 ? 2 : 3), bool kDedup = false>
__global__ void __launch_bounds__(kSegThreads, kMinB)
    segment_kernel(uint32_t* __restrict__ blocks, Geom g, const uint64_t* __restrict__ keys,
                   const uint16_t* __restrict__ boffs, uint64_t m, uint32_t groups, uint8_t* __restrict__ ans,
                   uint32_t per_cta, unsigned* __restrict__ work = nullptr, uint32_t items = 0, uint32_t rev = 0) {
  const uint64_t nchunks = (m + kPartChunk - 1) / kPartChunk;
  if constexpr (kDedup) {
    static_assert(kInsert, "the dedup table is for inserts");
    __shared__ uint64_t dtab[kDedupSlots];
    for (uint32_t e = threadIdx.x; e < kDedupSlots; e += kSegThreads) dtab[e] = e ^ 1u;
    __syncthreads();
    uint32_t b = blockIdx.x / groups;
    if (rev) b = gridDim.x / groups - 1 - b;
    const uint32_t grp = blockIdx.x % groups;
    const uint64_t c_begin = static_cast<uint64_t>(grp) * per_cta;
    const uint64_t c_end = c_begin + per_cta < nchunks ? c_begin + per_cta : nchunks;
    segment_item<kInsert, kSegQ, true>(blocks, g, keys, boffs, m, ans, b, c_begin, c_end, dtab);
    return;
  }
  if (!work) {
    // rev: this sweep runs the slices last-to-first (alternate sweeps do, so a
    // sweep starts on the slices the previous one left in L2)
    uint32_t b = blockIdx.x / groups;
    if (rev) b = gridDim.x / groups - 1 - b;
    const uint32_t grp = blockIdx.x % groups;
    const uint64_t c_begin = static_cast<uint64_t>(grp) * per_cta;
    const uint64_t c_end = c_begin + per_cta < nchunks ? c_begin + per_cta : nchunks;
    segment_item<kInsert, kSegQ>(blocks, g, keys, boffs, m, ans, b, c_begin, c_end);
    return;
  }
  __shared__ uint32_t next;
  for (;;) {
    if (threadIdx.x == 0) next = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t item = next;
    __syncthreads();
    if (item >= items) return;
    const uint32_t b = rev ? items / groups - 1 - item / groups : item / groups, grp = item % groups;
    const uint64_t c_begin = static_cast<uint64_t>(grp) * per_cta;
    const uint64_t c_end = c_begin + per_cta < nchunks ? c_begin + per_cta : nchunks;
    segment_item<kInsert, kSegQ>(blocks, g, keys, boffs, m, ans, b, c_begin, c_end);
  }
}

// Answers back to source order: one CTA per chunk reads the chunk's answer
// bytes and 16-bit positions (both contiguous), scatters them into shared
// memory and writes the chunk's result bits (ballot-packed) or bytes.
constexpr int kUnpermThreads = 256;

__global__ void __launch_bounds__(kUnpermThreads, 4) unpermute_kernel(const uint8_t* __restrict__ ans,
                                                                   const uint16_t* __restrict__ pos16, uint64_t m,
                                                                   void* __restrict__ out, bool bits,
                                                                   const uint16_t* __restrict__ boffs = nullptr) {
  static_assert(kPartChunk <= 65536, "positions are 16-bit");
  __shared__ __align__(16) uint8_t a[kPartChunk];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kPartChunk;
  // chunks laid out region by region (blocked_find_regions) carry their own
  // key count; otherwise every chunk but the last is full
  const uint32_t cnt = boffs ? boffs[static_cast<uint64_t>(blockIdx.x) * kBoffStride + kChunkBuckets]
                             : static_cast<uint32_t>(m - base < kPartChunk ? m - base : kPartChunk);
  if (cnt == kPartChunk) {
    // full chunk: 8 positions (16 B) + 8 answers (8 B) per vector load
    constexpr int kVec = kPartChunk / (kUnpermThreads * 8);
    uint4 pv[kVec];
    uint2 av[kVec];
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const uint32_t i = (k * kUnpermThreads + threadIdx.x) * 8;
      pv[k] = __ldg(reinterpret_cast<const uint4*>(pos16 + base + i));
      av[k] = __ldg(reinterpret_cast<const uint2*>(ans + base + i));
    }
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const uint32_t pw[4] = {pv[k].x, pv[k].y, pv[k].z, pv[k].w};
      const uint32_t aw[2] = {av[k].x, av[k].y};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        SBBF_DCHECK(((pw[e >> 1] >> ((e & 1) * 16)) & 0xffffu) < kPartChunk);
        a[(pw[e >> 1] >> ((e & 1) * 16)) & 0xffffu] = static_cast<uint8_t>(aw[e >> 2] >> ((e & 3) * 8));
      }
    }
  } else {
    for (uint32_t i = threadIdx.x; i < cnt; i += kUnpermThreads) {
      SBBF_DCHECK(pos16[base + i] < cnt);
      a[pos16[base + i]] = ans[base + i];
    }
  }
  __syncthreads();
  if (bits) {
    uint32_t* ob = static_cast<uint32_t*>(out) + (base >> 5);
    for (uint32_t wd = warp; wd * 32 < cnt; wd += kUnpermThreads / 32) {
      const uint32_t i = wd * 32 + lane;
      const uint32_t word = __ballot_sync(0xffffffffu, i < cnt && a[i]);
      if (lane == 0) ob[wd] = word;
    }
  } else {
    uint8_t* o = static_cast<uint8_t*>(out) + base;
    for (uint32_t i = threadIdx.x; i < cnt; i += kUnpermThreads) o[i] = a[i];
  }
}

// Full chunks of 16-byte aligned keys go through chunk_scatter_tma_kernel
// (config 4, ncu: 2^28-key lookup partition 0.98 -> 0.78 ms, 2^26-key insert
// partition 0.24 -> 0.18 ms; profiles/r2x_*). SBBF_SCATTER_TMA=0 selects the
// LSU kernel (A/B only).
bool scatter_tma() {
  static const bool on = [] {
    const char* v = getenv("SBBF_SCATTER_TMA");
    return !(v && v[0] == '0');
  }();
  return on;
}

// unpermute with the loads on the TMA engine: persistent CTAs, each chunk's
// positions (8 KB) and answer bytes (4 KB) bulk-loaded into one of two
// shared buffers while the previous chunk is scattered into source order.
// Full chunks only (the caller sends a partial last chunk through
// unpermute_kernel).
struct UnpermTmaSmem {
  alignas(16) uint16_t pos[2][kPartChunk];
  alignas(16) uint8_t ans[2][kPartChunk];
  alignas(16) uint8_t a[kPartChunk];
  alignas(8) uint64_t bar[2];
};

__global__ void __launch_bounds__(kUnpermThreads, 8)
    unpermute_tma_kernel(const uint8_t* __restrict__ ans, const uint16_t* __restrict__ pos16, uint64_t nfull,
                         void* __restrict__ out, bool bits) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  UnpermTmaSmem& sm = *reinterpret_cast<UnpermTmaSmem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kPosBytes = kPartChunk * sizeof(uint16_t), kAnsBytes = kPartChunk;
  auto issue = [&](uint64_t ch, uint32_t k) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&sm.bar[k])),
                 "r"(kPosBytes + kAnsBytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(sm.pos[k])),
                 "l"(pos16 + ch * kPartChunk), "r"(kPosBytes), "r"(smem_addr(&sm.bar[k]))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(sm.ans[k])),
                 "l"(ans + ch * kPartChunk), "r"(kAnsBytes), "r"(smem_addr(&sm.bar[k]))
                 : "memory");
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    if (blockIdx.x < nfull) issue(blockIdx.x, 0);
  }
  __syncthreads();
  uint32_t it = 0;
  for (uint64_t ch = blockIdx.x; ch < nfull; ch += gridDim.x, ++it) {
    const uint32_t k = it & 1;
    if (threadIdx.x == 0 && ch + gridDim.x < nfull) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(ch + gridDim.x, k ^ 1);
    }
    bulk_wait(&sm.bar[k], (it >> 1) & 1);
    constexpr int kVec = kPartChunk / (kUnpermThreads * 8);
#pragma unroll
    for (int v = 0; v < kVec; ++v) {
      const uint32_t i = (v * kUnpermThreads + threadIdx.x) * 8;
      const uint4 pv = *reinterpret_cast<const uint4*>(&sm.pos[k][i]);
      const uint2 av = *reinterpret_cast<const uint2*>(&sm.ans[k][i]);
      const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
      const uint32_t aw[2] = {av.x, av.y};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        SBBF_DCHECK(((pw[e >> 1] >> ((e & 1) * 16)) & 0xffffu) < kPartChunk);
        sm.a[(pw[e >> 1] >> ((e & 1) * 16)) & 0xffffu] = static_cast<uint8_t>(aw[e >> 2] >> ((e & 3) * 8));
      }
    }
    __syncthreads();
    const uint64_t base = ch * kPartChunk;
    if (bits) {
      uint32_t* ob = static_cast<uint32_t*>(out) + (base >> 5);
      for (uint32_t wd = warp; wd < kPartChunk / 32; wd += kUnpermThreads / 32) {
        const uint32_t word = __ballot_sync(0xffffffffu, sm.a[wd * 32 + lane] != 0);
        if (lane == 0) ob[wd] = word;
      }
    } else {
      uint4* o = reinterpret_cast<uint4*>(static_cast<uint8_t*>(out) + base);
      const uint4* src = reinterpret_cast<const uint4*>(sm.a);
      for (uint32_t v = threadIdx.x; v < kPartChunk / 16; v += kUnpermThreads) o[v] = src[v];
    }
    __syncthreads();
  }
}

// Full chunks go through unpermute_tma_kernel (config 4 lookups 103.3 ->
// 104.7 Gkeys/s, profiles/r2z_*); SBBF_UNPERM_TMA=0 selects unpermute_kernel
// (A/B only).
bool unperm_tma() {
  static const bool on = [] {
    const char* v = getenv("SBBF_UNPERM_TMA");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Answers of m keys (chunk layout) back to source order into `dst`.
cudaError_t launch_unpermute(const DeviceInfo& di, const uint8_t* ans, const uint16_t* pos16, uint64_t m, void* dst,
                             bool bits, cudaStream_t s) {
  KTime kt(kKUnpermute, s);
  const uint64_t nfull = m / kPartChunk;
  // byte output needs 16-byte aligned chunk rows; bit output 4-byte words
  const bool aligned = bits || (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  if (unperm_tma() && nfull && aligned) {
    static const cudaError_t attr = cudaFuncSetAttribute(
        unpermute_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(UnpermTmaSmem)));
    if (attr != cudaSuccess) return attr;
    // SBBF_UNPERM_CTAS (A/B only): resident CTAs per SM (28 KB smem each;
    // 8: 0.205 ms per 2^28-key round, 4: 0.214, profiles/r2_ab/r2aq_*)
    static const uint64_t per_sm = [] {
      const char* e = getenv("SBBF_UNPERM_CTAS");
      const int v = e ? atoi(e) : 0;
      return static_cast<uint64_t>(v > 0 && v <= 8 ? v : 8);
    }();
    const uint64_t cap = static_cast<uint64_t>(di.sms) * per_sm;
    note_launch();
    unpermute_tma_kernel<<<static_cast<unsigned>(nfull < cap ? nfull : cap), kUnpermThreads, sizeof(UnpermTmaSmem),
                           s>>>(ans, pos16, nfull, dst, bits);
    cudaError_t e = cudaGetLastError();
    const uint64_t done = nfull * kPartChunk;
    if (e != cudaSuccess || done == m) return e;
    note_launch();
    void* rest = bits ? static_cast<void*>(static_cast<uint32_t*>(dst) + done / 32)
                      : static_cast<void*>(static_cast<uint8_t*>(dst) + done);
    unpermute_kernel<<<1, kUnpermThreads, 0, s>>>(ans + done, pos16 + done, m - done, rest, bits);
    return cudaGetLastError();
  }
  note_launch();
  unpermute_kernel<<<static_cast<unsigned>((m + kPartChunk - 1) / kPartChunk), kUnpermThreads, 0, s>>>(ans, pos16, m,
                                                                                                        dst, bits);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// fused lookup sweep (packed staging, answers gathered in shared memory)
// ---------------------------------------------------------------------------
// The segment_kernel + unpermute pair moves 3 B/key of positions and answer
// bytes through HBM twice and relaunches per round. Here the partition stores
// packed slots (BucketMap::pack: slice-relative block, source position, low
// hash bits) and one persistent grid does the rest: every warp owns up to
// kFusedChunks chunks for the whole sweep, walks the slices in order over its
// chunks' runs, and sets the bit of each hit at its SOURCE position in the
// warp's shared-memory copy of those chunks' result bitmaps (one 512-byte row
// per chunk). When its runs are done it writes the rows out as the caller's
// bitmap words or bytes. No position array, no answer bytes, no unpermute
// launch; the warps free-run (equal work per slice keeps them within a slice
// or two of each other, so the keys in flight still share an L2-resident part
// of the filter).
constexpr int kFusedThreads = 256;
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr uint32_t kFusedChunks = 8;  // chunks per warp at most (6 CTAs/SM x 32 KB of bitmap rows)
constexpr uint32_t kRowWords = kPartChunk / 32;

struct FusedArgs {
  const uint32_t* blocks;
  const uint64_t* keys;   // packed slots, chunk layout
  const uint16_t* boffs;  // [nchunks][kBoffStride]
  void* out;              // bitmap words / bytes of this round, chunk ch at key ch * kPartChunk
  uint64_t nchunks;
  uint64_t nb_global, nb_local, mult;
  uint32_t S, bits, W, rev, sentinel, out_bits;
  // Slice pacing: CTAs count the sweep steps they finish in done[step]; a CTA
  // enters step k only when every CTA has finished step k - slack, so the
  // keys in flight span at most `slack` slices (free-running warps drift
  // apart and thrash L2: ncu, 8 CTAs/SM read the filter 5.4x per round).
  // Only a locality device: the wait is bounded and results never depend on
  // it. done == nullptr: free-running.
  unsigned* done;
  uint32_t slack;
};

__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
constexpr uint32_t kPaceMaxPolls = 1u << 13;  // ~4 ms at 500 ns per poll, then the CTA stops pacing

template <bool kTop, int kMinB>
__global__ void __launch_bounds__(kFusedThreads, kMinB) sweep_find_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(16) unsigned char fs_raw[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t W = a.W, S = a.S, T = S + 1;
  uint32_t* const rows = reinterpret_cast<uint32_t*>(fs_raw) + warp * W * kRowWords;  // [W][128] result bits
  uint64_t* const starts = reinterpret_cast<uint64_t*>(fs_raw + kFusedWarps * W * kRowWords * sizeof(uint32_t));
  uint16_t* const tab = reinterpret_cast<uint16_t*>(starts + (kTop ? 0 : S)) + warp * W * T;  // [W][S + 1] run offsets
  const uint32_t TW = gridDim.x * kFusedWarps, gw = blockIdx.x * kFusedWarps + warp;  // nchunks < 2^32
  const uint64_t pol = dev::policy_evict_first();  // lives in a uniform register (the load's descriptor)
  auto ld_slot = [&](const uint64_t* q) { return dev::ld_stream_u64(q, pol); };
  for (uint32_t k = lane; k < W * kRowWords; k += 32) rows[k] = 0;
  for (uint32_t i = 0; i < W; ++i) {
    const uint64_t ch = gw + static_cast<uint64_t>(i) * TW;
    for (uint32_t l = lane; l < T; l += 32) tab[i * T + l] = ch < a.nchunks ? a.boffs[ch * kBoffStride + l] : uint16_t{0};
  }
  if constexpr (!kTop) {
    for (uint32_t q = threadIdx.x; q < S; q += kFusedThreads) starts[q] = bucket_start(q, a.mult);
    __syncthreads();
  }
  __syncwarp();
  // run (bucket b, chunk row i) of this warp: first slot and length
  auto run_of = [&](uint32_t b, uint32_t i, uint32_t& len) -> const uint64_t* {
    const uint32_t st = tab[i * T + b], en = tab[i * T + b + 1];
    SBBF_DCHECK(st <= en && en <= kPartChunk);
    len = en - st;
    return a.keys + (gw + static_cast<uint64_t>(i) * TW) * kPartChunk + st + lane;
  };
  auto slice_first = [&](uint32_t b) -> uint64_t {
    if constexpr (kTop) return (static_cast<uint64_t>(b) * a.nb_global) >> a.bits;
    return starts[b];
  };
  // one probe step of a lane: the slot's sector on its way (a zero block for a key outside the shard)
  auto probe = [&](const uint32_t* slice, uint64_t h, dev::Block8& bl) {
    const uint32_t off = static_cast<uint32_t>(h >> 44);
    if (a.sentinel && off == kPackForeign) {
#pragma unroll
      for (int k = 0; k < 8; ++k) bl.w[k] = 0;
    } else {
      dev::ld_block_nc_normal(slice + static_cast<uint64_t>(off) * 8, bl);
    }
  };
  auto record = [&](uint32_t* row, const dev::Block8& bl, uint64_t h) {
    if (dev::block_contains(bl, h))
      atomicOr(row + (static_cast<uint32_t>(h >> 37) & (kRowWords - 1)), 1u << (static_cast<uint32_t>(h >> 32) & 31u));
  };
  __shared__ uint32_t pace_on;
  if (threadIdx.x == 0) pace_on = a.done != nullptr ? 1u : 0u;
  for (uint32_t bb = 0; bb < S; ++bb) {
    if (a.done) {
      // CTA-level pacing: the CTA has issued step bb - 1; it enters step bb once
      // every CTA has finished step bb - slack
      __syncthreads();
      if (threadIdx.x == 0) {
        if (bb > 0) atomicAdd(a.done + (bb - 1), 1u);
        if (pace_on && bb >= a.slack) {
          uint32_t polls = 0;
          while (ld_relaxed_gpu_u32(a.done + (bb - a.slack)) < gridDim.x && ++polls < kPaceMaxPolls) __nanosleep(500);
          if (polls >= kPaceMaxPolls) pace_on = 0;
        }
      }
      __syncthreads();
    }
    const uint32_t b = a.rev ? S - 1 - bb : bb;
    const uint32_t* const slice = a.blocks + slice_first(b) * 8;
    for (uint32_t i = 0; i < W; ++i) {
      uint32_t len;
      const uint64_t* p = run_of(b, i, len);
      uint32_t* const row = rows + i * kRowWords;
      uint64_t hn = lane < len ? ld_slot(p) : 0;
      for (uint32_t j = lane; j < len; j += 32, p += 32) {
        const uint64_t h = hn;
        dev::Block8 bl;
        probe(slice, h, bl);
        // the next step's slot loads while this step's sector is in flight
        if (j + 32 < len) hn = ld_slot(p + 32);
        record(row, bl, h);
      }
    }
  }
  __syncwarp();
  for (uint32_t r = 0; r < W; ++r) {
    const uint64_t ch = gw + static_cast<uint64_t>(r) * TW;
    if (ch >= a.nchunks) break;
    const uint64_t base = ch * kPartChunk;
    const uint32_t cnt = tab[r * T + S];  // the chunk's key count (end of its last run)
    const uint32_t* row = rows + r * kRowWords;
    if (a.out_bits) {
      uint32_t* ob = static_cast<uint32_t*>(a.out) + (base >> 5);
      for (uint32_t k = lane; k * 32 < cnt; k += 32) ob[k] = row[k];
    } else {
      uint8_t* o = static_cast<uint8_t*>(a.out) + base;
      const bool aligned = (reinterpret_cast<uintptr_t>(o) & 3) == 0;
      for (uint32_t k = lane; k * 4 < cnt; k += 32) {
        const uint32_t nib = (row[k >> 3] >> ((k & 7) * 4)) & 15u;
        const uint32_t v = (nib & 1u) | (nib & 2u) << 7 | (nib & 4u) << 14 | (nib & 8u) << 21;
        if (aligned && k * 4 + 4 <= cnt) {
          *reinterpret_cast<uint32_t*>(o + k * 4) = v;
        } else {
          for (uint32_t e = 0; e < 4 && k * 4 + e < cnt; ++e) o[k * 4 + e] = static_cast<uint8_t>(v >> (8 * e));
        }
      }
    }
  }
}

// SBBF_FIND_FUSED=0 selects the partition + segment_kernel + unpermute lookups (A/B only).
bool find_fused() {
  static const bool on = [] {
    const char* v = getenv("SBBF_FIND_FUSED");
    return !(v && v[0] == '0');
  }();
  return on;
}
// SBBF_FUSED_VARIANT (A/B only): 0 = 6 CTAs/SM (default), 1 = 8 CTAs/SM. Config 4
// lookups 105.8 vs 103.1 Gkeys/s; two sectors in flight per lane at 5 / 4
// CTAs/SM measured 101.5 / 100.8 (profiles/r2_ab/r2cl_*).
int fused_variant() {
  static const int v = [] {
    const char* e = getenv("SBBF_FUSED_VARIANT");
    const int x = e ? atoi(e) : 0;
    return x >= 0 && x <= 3 ? x : 0;
  }();
  return v;
}

// SBBF_FUSED_SLACK (A/B only): slices the sweep's warps may span (0 = free-running).
uint32_t fused_slack() {
  static const uint32_t v = [] {
    const char* e = getenv("SBBF_FUSED_SLACK");
    const int x = e ? atoi(e) : 2;
    return static_cast<uint32_t>(x >= 0 && x <= 8 ? x : 2);
  }();
  return v;
}
// SBBF_FUSED_W (A/B only): chunks per warp per round (1..kFusedChunks).
uint32_t fused_chunks() {
  static const uint32_t v = [] {
    const char* e = getenv("SBBF_FUSED_W");
    const int x = e ? atoi(e) : 0;
    return static_cast<uint32_t>(x >= 1 && x <= static_cast<int>(kFusedChunks) ? x : kFusedChunks);
  }();
  return v;
}

// Can this map's slots be packed (every slice within kPackOffBits of blocks)?
// `trusted`: no key of the batch lies outside the map's block range.
bool pack_map(BucketMap& bm, bool trusted) {
  const uint64_t limit = uint64_t{1} << kPackOffBits;
  bm.pack = 0;
  bm.pack_shift = 0;
  bm.sentinel = 0;
  if (bm.top_bits) {
    const uint64_t nb = bm.nb_global;
    if ((nb & (nb - 1)) == 0) {
      uint32_t lg = 0;
      while ((uint64_t{1} << lg) < nb) ++lg;
      if (lg <= bm.bits || lg - bm.bits > static_cast<uint32_t>(kPackOffBits)) return false;
      bm.pack_shift = 64 - (lg - bm.bits);
    } else if ((nb >> bm.bits) + 2 > limit) {
      return false;
    }
    bm.pack = 1;
    return true;
  }
  if (bm.mult == 0) return false;
  const uint32_t sentinel = trusted ? 0u : 1u;
  for (uint32_t q = 0; q < bm.S; ++q) {
    const uint64_t lo = bucket_start(q, bm.mult);
    const uint64_t hi = q + 1 < bm.S ? bucket_start(q + 1, bm.mult) : bm.nb_local;
    if (hi > lo && hi - lo > limit - sentinel) return false;
  }
  bm.pack = 1;
  bm.sentinel = sentinel;
  return true;
}

template <int BITS, bool kTop>
cudaError_t chunk_partition_bits(const DeviceInfo& di, const BucketMap& bm, const uint64_t* hashes, uint64_t m,
                                 uint64_t* out, uint16_t* pos16, uint16_t* boffs, cudaStream_t s) {
  static const cudaError_t attr = cudaFuncSetAttribute(
      chunk_scatter_kernel<BITS, kTop>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(ChunkSmem)));
  if (attr != cudaSuccess) return attr;
  if (scatter_tma() && (reinterpret_cast<uintptr_t>(hashes) & 15) == 0 && m >= kPartChunk) {
    static const cudaError_t attr_t =
        cudaFuncSetAttribute(chunk_scatter_tma_kernel<BITS, kTop>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(ChunkTmaSmem)));
    if (attr_t != cudaSuccess) return attr_t;
    const uint64_t nfull = m / kPartChunk;
    const uint64_t cap = static_cast<uint64_t>(di.sms) * kPartMinBlocks;
    note_launch();
    chunk_scatter_tma_kernel<BITS, kTop><<<static_cast<unsigned>(nfull < cap ? nfull : cap), kPartThreads,
                                           sizeof(ChunkTmaSmem), s>>>(hashes, nfull, bm, out, pos16, boffs);
    cudaError_t e = cudaGetLastError();
    const uint64_t done = nfull * kPartChunk;
    if (e != cudaSuccess || done == m) return e;
    note_launch();  // the partial last chunk
    chunk_scatter_kernel<BITS, kTop><<<1, kPartThreads, sizeof(ChunkSmem), s>>>(
        hashes + done, m - done, bm, out + done, pos16 ? pos16 + done : nullptr, boffs + nfull * kBoffStride);
    return cudaGetLastError();
  }
  const uint64_t nchunks = (m + kPartChunk - 1) / kPartChunk;
  // SBBF_PART_PER_SM (A/B only): partition CTAs per SM
  static const uint64_t per_sm = [] {
    const char* e = getenv("SBBF_PART_PER_SM");
    const int v = e ? atoi(e) : 0;
    return static_cast<uint64_t>(v > 0 ? v : kPartMinBlocks);
  }();
  const uint64_t grid = nchunks < static_cast<uint64_t>(di.sms) * per_sm ? nchunks
                                                                         : static_cast<uint64_t>(di.sms) * per_sm;
  note_launch();
  chunk_scatter_kernel<BITS, kTop><<<static_cast<unsigned>(grid), kPartThreads, sizeof(ChunkSmem), s>>>(
      hashes, m, bm, out, pos16, boffs);
  return cudaGetLastError();
}

cudaError_t chunk_partition(const DeviceInfo& di, const Geom& g, uint32_t S, const uint64_t* hashes, uint64_t m,
                            uint64_t* out, uint16_t* pos16, uint16_t* boffs, cudaStream_t s,
                            const BucketMap* packed = nullptr) {
  KTime kt(kKPartition, s);
  const BucketMap bm = packed ? *packed : make_map(g, S);
  switch (bm.bits * 2 + (bm.top_bits ? 1 : 0)) {
#define SBBF_CHUNK_CASE(B)                                                                  \
  case 2 * B:                                                                               \
    return chunk_partition_bits<B, false>(di, bm, hashes, m, out, pos16, boffs, s);         \
  case 2 * B + 1:                                                                           \
    return chunk_partition_bits<B, true>(di, bm, hashes, m, out, pos16, boffs, s);
    SBBF_CHUNK_CASE(1)
    SBBF_CHUNK_CASE(2)
    SBBF_CHUNK_CASE(3)
    SBBF_CHUNK_CASE(4)
    SBBF_CHUNK_CASE(5)
    SBBF_CHUNK_CASE(6)
    SBBF_CHUNK_CASE(7)
#undef SBBF_CHUNK_CASE
    default: return cudaErrorInvalidValue;
  }
}

// The persistent segment grid measured neutral on config 4 (profiles/r2p_*:
// the filter is read 1.3x instead of 3x, but the sweep is latency-bound, not
// DRAM-bound), so the one-shot grid stays the default (A/B only):
// SBBF_SEG_PERSIST=1 selects it for both phases, =2 for lookups only.
bool seg_persist(bool insert) {
  static const int on = [] {
    const char* v = getenv("SBBF_SEG_PERSIST");
    return v ? atoi(v) : 0;
  }();
  return on == 1 || (on == 2 && !insert);
}

// SBBF_SEG_INS_Q (A/B only): segments per warp step of the insert segment
// kernel (2 = default, 4, 8). Config 4 inserts (profiles/r2_ab/r2ax_*, r2ay_*):
// 2 segments x 16 chunks per CTA 57.1 Gkeys/s, 4 x 32 56.2, 4 x 64 55.4,
// 8 x 64 54.1, 1 x 16 54.2. Measured and removed (profiles/r2_ab): plain
// reds without the test load (8.5 Gkeys/s on config 4: the hot keys' reds
// serialise at L2), .cg / .nc test loads, an L2 prefetch of the next step's
// lines, bulk prefetch of the slice ahead, 4 CTAs/SM at 64 registers.
int seg_ins_q() {
  static const int v = [] {
    const char* e = getenv("SBBF_SEG_INS_Q");
    const int x = e ? atoi(e) : 2;
    return (x == 4 || x == 8) ? x : 2;
  }();
  return v;
}

// SBBF_SEG_DEDUP (A/B): 1 = the insert sweep skips hashes its CTA already
// ORed (shared-memory table) instead of test-loading each key's lane pair.
bool seg_dedup() {
  static const bool on = [] {
    const char* v = getenv("SBBF_SEG_DEDUP");
    return v && v[0] == '1';
  }();
  return on;
}

template <bool kInsert>
cudaError_t launch_segments(uint32_t* blocks, const Geom& g, const uint64_t* keys, const uint16_t* boffs, uint32_t S,
                            uint64_t m, uint8_t* ans, cudaStream_t s, unsigned* work = nullptr,
                            const DeviceInfo* di = nullptr, bool* flip = nullptr) {
  KTime kt(kInsert ? kKInsertSweep : kKProbe, s);
  // alternate the sweep direction per handle (SBBF_SEG_ALTERNATE=0 disables it: A/B only)
  static const bool alt = [] {
    const char* v = getenv("SBBF_SEG_ALTERNATE");
    return !(v && v[0] == '0');
  }();
  uint32_t rev = 0;
  if (flip && alt) {
    rev = *flip ? 1u : 0u;
    *flip = !*flip;
  }
  const uint64_t nchunks = (m + kPartChunk - 1) / kPartChunk;
  const bool persist = work && di && seg_persist(kInsert);
  const uint32_t per_cta = persist ? seg_items_chunks() : seg_chunks_per_cta(kInsert);
  const uint32_t groups = static_cast<uint32_t>((nchunks + per_cta - 1) / per_cta);
  if (persist) {
    const uint32_t items = S * groups;
    auto kern = kInsert ? segment_kernel<true, 4> : segment_kernel<false, 1, 8>;
    static const int occ_i = [] {
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, segment_kernel<true, 4>, kSegThreads, 0);
      return b > 0 ? b : 1;
    }();
    static const int occ_l = [] {
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, segment_kernel<false, 1, 8>, kSegThreads, 0);
      return b > 0 ? b : 1;
    }();
    uint64_t grid = static_cast<uint64_t>(di->sms) * (kInsert ? occ_i : occ_l);
    if (grid > items) grid = items;
    cudaError_t e = cudaMemsetAsync(work, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    note_launch();
    kern<<<static_cast<unsigned>(grid), kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta, work,
                                                               items, rev);
    return cudaGetLastError();
  }
  note_launch();
  // Segments per warp step / min CTAs per SM, measured on config 4: inserts
  // 2 / 4 at 16 chunks per CTA (seg_ins_q); lookups 1 / 8 — 1.54 ms per 2^28
  // keys, vs 1.82 (2 segments), 1.89 (4), 2.37 (8): occupancy beats per-lane
  // MLP (profiles/r1_blocked_partition.md; round 2: 2 segments at 8 CTAs/SM
  // spill and reach 86 vs 104 Gkeys/s).
  const unsigned grid = S * groups;
  if constexpr (kInsert) {
    const int q = seg_ins_q();
    if (seg_dedup()) {
      if (q == 4)
        segment_kernel<true, 4, 3, true><<<grid, kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta,
                                                                      nullptr, 0u, rev);
      else
        segment_kernel<true, 2, 4, true><<<grid, kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta,
                                                                      nullptr, 0u, rev);
    } else if (q == 4)
      segment_kernel<true, 4><<<grid, kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta, nullptr, 0u,
                                                           rev);
    else if (q == 8)
      segment_kernel<true, 8><<<grid, kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta, nullptr, 0u,
                                                           rev);
    else
      segment_kernel<true, 2, 4><<<grid, kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta, nullptr,
                                                              0u, rev);
  } else {
    segment_kernel<false, 1, 8><<<grid, kSegThreads, 0, s>>>(blocks, g, keys, boffs, m, groups, ans, per_cta, nullptr,
                                                             0u, rev);
  }
  return cudaGetLastError();
}

struct Scratch {
  bool* flip = nullptr;  // the handle's sweep-direction toggle (arena mode)
  uint64_t* keys = nullptr;
  uint16_t* boffs = nullptr;
  uint16_t* pos16 = nullptr;
  uint8_t* ans = nullptr;
  unsigned* work = nullptr;  // persistent segment grid's work counter
  uint64_t* keys2 = nullptr;  // tile inserts: keys grouped by tile
  uint32_t* runs = nullptr;   // tile inserts: run starts per (slice, group, tile)
  bool pooled = false;  // from the stream-ordered pool (freed per call) rather than the handle's arena
};

// tile_scatter CTAs per slice for a batch chunk of cap keys, and the run table's entries
uint64_t tile_groups(uint64_t cap) {
  const uint64_t nchunks = (cap + kPartChunk - 1) / kPartChunk;
  return (nchunks + kTileGroupChunks - 1) / kTileGroupChunks;
}
uint64_t tile_runs_entries(uint64_t cap) { return 128 * tile_groups(cap) * (kTilesPerSlice + 1); }

uint64_t align256(uint64_t b) { return (b + 255) & ~uint64_t{255}; }

uint64_t scratch_bytes(uint64_t cap, bool lookup) {
  const uint64_t nchunks = (cap + kPartChunk - 1) / kPartChunk;
  return align256(cap * sizeof(uint64_t)) + align256(nchunks * kBoffStride * sizeof(uint16_t)) +
         (lookup ? align256(cap * sizeof(uint16_t)) + align256(cap)
                 : align256(cap * sizeof(uint64_t)) + align256(tile_runs_entries(cap) * sizeof(uint32_t))) +
         align256(kChunkBuckets * sizeof(unsigned));
}

}  // namespace

// Per-handle blocked-path context: a scratch arena that persists across calls
// (one cudaMalloc, grown on demand; the stream-ordered pool's trimming and
// growth inside timed steps is what produced the occasional 10x config-4
// step), ordered across callers' streams by an `idle` event. Calls being
// captured into a CUDA graph take their scratch from the stream-ordered pool
// instead (graph-safe).
struct BlockedCtx {
  std::mutex mu;
  char* base = nullptr;
  uint64_t cap = 0;
  cudaEvent_t idle = nullptr;
  bool flip = false;  // direction of the next segment sweep
  cudaError_t init() {  // under mu
    if (idle) return cudaSuccess;
    return cudaEventCreateWithFlags(&idle, cudaEventDisableTiming);
  }
  ~BlockedCtx() {
    if (idle) cudaEventSynchronize(idle);
    cudaFree(base);
    if (idle) cudaEventDestroy(idle);
  }
};

BlockedCtx* blocked_ctx_create() { return new (std::nothrow) BlockedCtx; }
void blocked_ctx_destroy(BlockedCtx* c) { delete c; }
int blocked_ctx_release(BlockedCtx* c) {
  if (!c) return 0;
  std::lock_guard<std::mutex> lock(c->mu);
  if (c->idle) cudaEventSynchronize(c->idle);
  cudaFree(c->base);
  c->base = nullptr;
  c->cap = 0;
  return 0;
}

namespace {

// One blocked call's hold on the handle's context: the lock (one call at a
// time enqueues), the arena sized for `need` bytes and ordered behind the
// previous call's use (its `idle` event), released by recording `idle` on s.
class CallScope {
 public:
  CallScope(BlockedCtx* ctx, cudaStream_t s, uint64_t need) : ctx_(ctx), s_(s) {
    if (!ctx_) return;
    lock_ = std::unique_lock<std::mutex>(ctx_->mu);
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      capturing_ = true;
      return;
    }
    err_ = ctx_->init();
    if (err_ != cudaSuccess) return;
    if (ctx_->cap < need) {
      if (ctx_->base) {
        cudaEventSynchronize(ctx_->idle);
        cudaFree(ctx_->base);
        ctx_->base = nullptr;
        ctx_->cap = 0;
      }
      err_ = cudaMalloc(reinterpret_cast<void**>(&ctx_->base), need);
      if (err_ != cudaSuccess) {
        ctx_->base = nullptr;
        return;
      }
      ctx_->cap = need;
    }
    err_ = cudaStreamWaitEvent(s, ctx_->idle, 0);  // the previous caller is done with the arena
    arena_ = err_ == cudaSuccess;
  }
  ~CallScope() {
    if (arena_) cudaEventRecord(ctx_->idle, s_);
  }
  bool arena() const { return arena_; }
  bool capturing() const { return capturing_; }
  cudaError_t error() const { return err_; }
  BlockedCtx* ctx() const { return ctx_; }
  // carve `bytes` of the arena (arena mode) at the running offset
  char* take(uint64_t bytes) {
    char* p = ctx_->base + used_;
    used_ += align256(bytes);
    return p;
  }

 private:
  BlockedCtx* ctx_;
  cudaStream_t s_;
  std::unique_lock<std::mutex> lock_;
  bool arena_ = false, capturing_ = false;
  cudaError_t err_ = cudaSuccess;
  uint64_t used_ = 0;
};

cudaError_t alloc_scratch(Scratch& sc, uint64_t cap, bool lookup, cudaStream_t s, CallScope* scope = nullptr) {
  const uint64_t nchunks = (cap + kPartChunk - 1) / kPartChunk;
  if (scope && scope->arena()) {
    sc.keys = reinterpret_cast<uint64_t*>(scope->take(cap * sizeof(uint64_t)));
    sc.boffs = reinterpret_cast<uint16_t*>(scope->take(nchunks * kBoffStride * sizeof(uint16_t)));
    if (lookup) {
      sc.pos16 = reinterpret_cast<uint16_t*>(scope->take(cap * sizeof(uint16_t)));
      sc.ans = reinterpret_cast<uint8_t*>(scope->take(cap));
    } else {
      sc.keys2 = reinterpret_cast<uint64_t*>(scope->take(cap * sizeof(uint64_t)));
      sc.runs = reinterpret_cast<uint32_t*>(scope->take(tile_runs_entries(cap) * sizeof(uint32_t)));
    }
    sc.work = reinterpret_cast<unsigned*>(scope->take(kChunkBuckets * sizeof(unsigned)));
    sc.flip = &scope->ctx()->flip;
    sc.pooled = false;
    return cudaSuccess;
  }
  retain_pool();
  sc.pooled = true;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sc.keys), cap * sizeof(uint64_t), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&sc.boffs), nchunks * kBoffStride * sizeof(uint16_t), s);
  if (lookup && e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&sc.pos16), cap * sizeof(uint16_t), s);
  if (lookup && e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&sc.ans), cap, s);
  if (!lookup && e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&sc.keys2), cap * sizeof(uint64_t), s);
  if (!lookup && e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&sc.runs), tile_runs_entries(cap) * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&sc.work), kChunkBuckets * sizeof(unsigned), s);
  return e;
}

void free_scratch(Scratch& sc, cudaStream_t s) {
  if (sc.pooled) {
    if (sc.keys) cudaFreeAsync(sc.keys, s);
    if (sc.boffs) cudaFreeAsync(sc.boffs, s);
    if (sc.pos16) cudaFreeAsync(sc.pos16, s);
    if (sc.ans) cudaFreeAsync(sc.ans, s);
    if (sc.work) cudaFreeAsync(sc.work, s);
    if (sc.keys2) cudaFreeAsync(sc.keys2, s);
    if (sc.runs) cudaFreeAsync(sc.runs, s);
  }
  sc = Scratch{};
}

}  // namespace

cudaError_t shard_partition(const DeviceInfo& di, uint64_t total, uint32_t parts, const uint64_t* d_bounds,
                            const uint64_t* hashes, uint64_t n, uint64_t* d_counts, uint64_t* d_cursor,
                            uint64_t* d_out, uint32_t* d_pos, cudaStream_t s) {
  if (n == 0) return cudaMemsetAsync(d_counts, 0, parts * sizeof(uint64_t), s);
  const Geom whole{total, 0, total};
  return bucket_partition(di, whole, parts, hashes, n, d_counts, d_cursor, d_out, d_pos, s, d_bounds);
}

cudaError_t route_partition(const DeviceInfo& di, uint64_t total, uint32_t parts, const uint64_t* d_bounds,
                            const uint64_t* hashes, uint64_t n, uint64_t* d_counts, uint32_t* d_pos,
                            uint64_t* const* d_dst, unsigned long long* const* d_count_dst, cudaStream_t s) {
  const Geom whole{total, 0, total};
  RouteOut route;
  route.dst = d_dst;
  route.count_dst = d_count_dst;
  return bucket_partition(di, whole, parts, hashes, n, d_counts, nullptr, nullptr, d_pos, s, d_bounds, route);
}

namespace {

// One batch chunk (m <= blocked_round() keys) through the single-level path.
// Tile inserts (tile_scatter_kernel / tile_apply_persistent_kernel) apply to whole
// power-of-two filters of 2^20..2^26 blocks (32 MiB - 2 GiB): S = nb / 2^19
// slices of 256 tiles of 2048 blocks, slice = the hash's top bits.
// SBBF_INSERT_TILES=0 selects the segment sweep (A/B only).
uint32_t tile_slices(const Geom& g, uint64_t m, const Scratch& sc) {
  static const bool on = [] {
    const char* v = getenv("SBBF_INSERT_TILES");
    return v && v[0] == '1';
  }();
  const uint64_t nb = g.nb_global;
  if (!on || !sc.keys2 || !sc.runs || g.first != 0 || g.nb_local != nb || (nb & (nb - 1)) != 0) return 0;
  if (nb < (uint64_t{1} << 20) || nb > (uint64_t{1} << 26) || tile_groups(m) > kTileMaxGroups) return 0;
  return static_cast<uint32_t>(nb >> (kTileBits + kTileLog2));
}

cudaError_t insert_tiles(const DeviceInfo& di, uint32_t* blocks, const Geom& g, uint32_t S, const uint64_t* keys,
                         uint64_t m, Scratch& sc, cudaStream_t s) {
  cudaError_t e = chunk_partition(di, g, S, keys, m, sc.keys, nullptr, sc.boffs, s);
  if (e != cudaSuccess) return e;
  static const cudaError_t a1 = cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     static_cast<int>(sizeof(TileScatterSmem)));
  static const cudaError_t a2 =
      cudaFuncSetAttribute(tile_apply_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(TileApply2Smem)));
  if (a1 != cudaSuccess) return a1;
  if (a2 != cudaSuccess) return a2;
  const uint32_t groups = static_cast<uint32_t>(tile_groups(m));
  KTime kt(kKTile, s);
  note_launch();
  tile_scatter_kernel<<<S * groups, kTileScatterThreads, sizeof(TileScatterSmem), s>>>(g.nb_global, S, sc.keys,
                                                                                       sc.boffs, m, groups, sc.keys2,
                                                                                       sc.runs);
  uint32_t rev = 0;
  if (sc.flip) {
    rev = *sc.flip ? 1u : 0u;
    *sc.flip = !*sc.flip;
  }
  note_launch();
  const uint32_t ntiles = S * kTilesPerSlice;
  tile_apply_persistent_kernel<<<static_cast<unsigned>(ntiles < static_cast<uint32_t>(di.sms) ? ntiles : di.sms),
                                 kTileP2Threads, sizeof(TileApply2Smem), s>>>(blocks, g.nb_global, S, sc.keys2, sc.runs,
                                                                              groups, rev);
  return cudaGetLastError();
}

cudaError_t insert_chunk(const DeviceInfo& di, uint32_t* blocks, const Geom& g, uint32_t parts, const uint64_t* keys,
                         uint64_t m, Scratch& sc, cudaStream_t s) {
  if (const uint32_t S = tile_slices(g, m, sc)) return insert_tiles(di, blocks, g, S, keys, m, sc, s);
  cudaError_t e = chunk_partition(di, g, parts, keys, m, sc.keys, nullptr, sc.boffs, s);
  if (e == cudaSuccess)
    e = launch_segments<true>(blocks, g, sc.keys, sc.boffs, parts, m, nullptr, s, sc.work, &di, sc.flip);
  return e;
}

// The fused sweep's launch shape for a map: the kernel, how many chunks one
// launch can take (resident warps x chunks per warp) and the dynamic smem.
struct FusedShape {
  void (*kern)(const FusedArgs) = nullptr;
  uint64_t max_ctas = 0;
  uint32_t Wmax = 0;
  bool top = false;
  uint32_t S = 0;
  size_t smem(uint32_t W) const {
    return static_cast<size_t>(kFusedWarps) * W * kRowWords * sizeof(uint32_t) + (top ? 0 : S * sizeof(uint64_t)) +
           static_cast<size_t>(kFusedWarps) * W * (S + 1) * sizeof(uint16_t);
  }
  uint64_t max_chunks() const { return max_ctas * kFusedWarps * Wmax; }
};

template <bool kTop>
cudaError_t fused_shape_for(const DeviceInfo& di, const BucketMap& bm, FusedShape& fs) {
  using Kern = void (*)(const FusedArgs);
  static const Kern kerns[2] = {sweep_find_kernel<kTop, 6>, sweep_find_kernel<kTop, 8>};
  static const int kern_ctas[2] = {6, 8};
  static const cudaError_t attr = [] {
    cudaError_t r = cudaSuccess;
    for (Kern k : kerns)
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    for (Kern k : kerns)
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    return r;
  }();
  if (attr != cudaSuccess) return attr;
  fs.kern = kerns[fused_variant()];
  fs.top = kTop;
  fs.S = bm.S;
  // chunks per warp: as many as keep the kernel's register-limited occupancy
  // (a round sweeps the whole filter once, so its cost per key falls with W)
  const int want = kern_ctas[fused_variant()];
  int occ = 0;
  for (fs.Wmax = fused_chunks();; --fs.Wmax) {
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fs.kern, kFusedThreads, fs.smem(fs.Wmax));
    if (e != cudaSuccess) return e;
    if (occ >= want || fs.Wmax == 1) break;
  }
  if (occ < 1) return cudaErrorNotSupported;
  fs.max_ctas = static_cast<uint64_t>(di.sms) * occ;
  return cudaSuccess;
}

cudaError_t fused_shape(const DeviceInfo& di, const BucketMap& bm, FusedShape& fs) {
  return bm.top_bits ? fused_shape_for<true>(di, bm, fs) : fused_shape_for<false>(di, bm, fs);
}

// One sweep over nchunks <= fs.max_chunks() staged chunks (packed slots in
// sc.keys, run offsets in sc.boffs); `out` takes chunk ch's answers at key
// ch * kPartChunk (bitmap words or bytes).
cudaError_t fused_sweep(const FusedShape& fs, const uint32_t* blocks, const Geom& g, const BucketMap& bm, Scratch& sc,
                        uint64_t nchunks, void* out, bool bits, cudaStream_t s) {
  KTime kt(kKProbe, s);
  FusedArgs a;
  a.blocks = blocks;
  a.keys = sc.keys;
  a.boffs = sc.boffs;
  a.out = out;
  a.nchunks = nchunks;
  a.nb_global = g.nb_global;
  a.nb_local = g.nb_local;
  a.mult = bm.mult;
  a.S = bm.S;
  a.bits = bm.bits;
  a.W = static_cast<uint32_t>((nchunks + fs.max_ctas * kFusedWarps - 1) / (fs.max_ctas * kFusedWarps));
  a.rev = 0;
  if (sc.flip) {  // alternate the sweep direction: a sweep starts on the slices the last one left in L2
    a.rev = *sc.flip ? 1u : 0u;
    *sc.flip = !*sc.flip;
  }
  a.sentinel = bm.sentinel;
  a.out_bits = bits ? 1u : 0u;
  a.done = sc.work;
  a.slack = fused_slack();
  if (a.done && a.slack) {
    const cudaError_t e = cudaMemsetAsync(a.done, 0, kChunkBuckets * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
  } else {
    a.done = nullptr;
  }
  const uint64_t grid = (nchunks + static_cast<uint64_t>(kFusedWarps) * a.W - 1) / (kFusedWarps * a.W);
  note_launch();
  fs.kern<<<static_cast<unsigned>(grid), kFusedThreads, fs.smem(a.W), s>>>(a);
  return cudaGetLastError();
}

// Fused lookups of m keys: rounds of up to fs.max_chunks() chunks, each a
// packed partition and one persistent sweep.
cudaError_t find_chunk_fused(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const BucketMap& bm,
                             const uint64_t* keys, uint64_t m, Scratch& sc, uint64_t scratch_keys, void* dst, bool bits,
                             cudaStream_t s) {
  FusedShape fs;
  cudaError_t e = fused_shape(di, bm, fs);
  if (e != cudaSuccess) return e;
  uint64_t round = fs.max_chunks() * kPartChunk;
  if (round > scratch_keys) round = scratch_keys / kPartChunk * kPartChunk;  // the scratch holds one round
  if (round == 0) return cudaErrorNotSupported;
  static const bool dbg = getenv("SBBF_FUSED_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "[sbbf] fused sweep: %llu CTAs, %llu keys per round, S=%u\n",
                   static_cast<unsigned long long>(fs.max_ctas), static_cast<unsigned long long>(round), bm.S);
  for (uint64_t off = 0; e == cudaSuccess && off < m; off += round) {
    const uint64_t mm = m - off < round ? m - off : round;
    e = chunk_partition(di, g, bm.S, keys + off, mm, sc.keys, nullptr, sc.boffs, s, &bm);
    if (e == cudaSuccess)
      e = fused_sweep(fs, blocks, g, bm, sc, (mm + kPartChunk - 1) / kPartChunk,
                      bits ? static_cast<void*>(static_cast<uint32_t*>(dst) + off / 32)
                           : static_cast<void*>(static_cast<uint8_t*>(dst) + off),
                      bits, s);
  }
  return e;
}

// The fused lookup of m keys (any number of rounds; the scratch holds
// scratch_keys slots), or cudaErrorNotSupported when the map cannot be packed.
// `dense_only` (AUTO dispatch): batches thinner than a key per block keep the
// unfused kernels — their one-shot grid copes better with runs of a few keys
// (config 5's world-1 sample, 0.5 keys per block: 31.3 vs 28.5 Gkeys/s).
cudaError_t try_find_fused(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, uint32_t parts,
                           const uint64_t* keys, uint64_t m, Scratch& sc, uint64_t scratch_keys, void* dst, bool bits,
                           cudaStream_t s, bool trusted, bool dense_only) {
  if (!find_fused() || (dense_only && m < g.nb_local)) return cudaErrorNotSupported;
  BucketMap bm = make_map(g, parts);
  if (!pack_map(bm, trusted)) return cudaErrorNotSupported;
  const cudaError_t e = find_chunk_fused(di, blocks, g, bm, keys, m, sc, scratch_keys, dst, bits, s);
  if (e == cudaErrorNotSupported) cudaGetLastError();
  return e;
}

cudaError_t find_chunk(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, uint32_t parts,
                       const uint64_t* keys, uint64_t m, Scratch& sc, void* dst, bool bits, cudaStream_t s,
                       bool trusted = false, bool dense_only = false) {
  {
    const cudaError_t ef = try_find_fused(di, blocks, g, parts, keys, m, sc, m, dst, bits, s, trusted, dense_only);
    if (ef != cudaErrorNotSupported) return ef;
  }
  // 1. every chunk bucket-major in its own region (+ positions, offsets)
  cudaError_t e = chunk_partition(di, g, parts, keys, m, sc.keys, sc.pos16, sc.boffs, s);
  // 2. probe slice by slice (L2-resident), one answer byte per routed slot
  if (e == cudaSuccess)
    e = launch_segments<false>(const_cast<uint32_t*>(blocks), g, sc.keys, sc.boffs, parts, m, sc.ans, s, sc.work, &di,
                                  sc.flip);
  // 3. back to source order, straight into the caller's bitmap / bytes
  if (e == cudaSuccess) {
    e = launch_unpermute(di, sc.ans, sc.pos16, m, dst, bits, s);
  }
  return e;
}

// Filters beyond kChunkBuckets slices (> 4 GiB): a first partition groups the
// batch chunk by "super-slice" (exact block ranges, global bucket-major
// layout with source positions), then each super-slice runs the single-level
// path on its sub-filter, so every slice the probes touch stays ~32 MiB.
struct TwoLevel {
  uint64_t* keys = nullptr;       // [m] grouped by super-slice
  uint32_t* pos = nullptr;        // [m] source index (lookups)
  uint8_t* ans = nullptr;         // [m] answers in grouped order (lookups)
  uint8_t* bytes = nullptr;       // [m] answers in source order (bit output)
  uint64_t* counts = nullptr;     // [2 * S]
};

cudaError_t super_counts(const DeviceInfo& di, const Geom& g, const BlockedPlan& plan, const uint64_t* keys,
                         uint64_t m, TwoLevel& tl, bool lookup, cudaStream_t s, std::vector<uint64_t>& h) {
  cudaError_t e = bucket_partition(di, g, plan.super_parts, keys, m, tl.counts, tl.counts + plan.super_parts, tl.keys,
                                   lookup ? tl.pos : nullptr, s, plan.d_super_bounds);
  h.assign(plan.super_parts, 0);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h.data(), tl.counts, plan.super_parts * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}

Geom sub_geom(const Geom& g, const std::vector<uint64_t>& sb, uint32_t k) {
  return Geom{g.nb_global, g.first + sb[k], sb[k + 1] - sb[k]};
}

}  // namespace

cudaError_t blocked_insert(const DeviceInfo& di, uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                           const uint64_t* hashes, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t cap = n < blocked_round() ? n : blocked_round();
  Scratch sc;
  TwoLevel tl;
  const bool two = plan.super_parts > 1;
  CallScope scope(plan.ctx, s, scratch_bytes(cap, false));
  if (scope.error() != cudaSuccess) return scope.error();
  cudaError_t e = alloc_scratch(sc, cap, false, s, &scope);
  if (e == cudaSuccess && two) e = cudaMallocAsync(reinterpret_cast<void**>(&tl.keys), cap * sizeof(uint64_t), s);
  if (e == cudaSuccess && two)
    e = cudaMallocAsync(reinterpret_cast<void**>(&tl.counts), 2 * plan.super_parts * sizeof(uint64_t), s);
  std::vector<uint64_t> cnt;
  for (uint64_t off = 0; e == cudaSuccess && off < n; off += cap) {
    const uint64_t m = n - off < cap ? n - off : cap;
    if (!two) {
      e = insert_chunk(di, blocks, g, plan.parts, hashes + off, m, sc, s);
      continue;
    }
    e = super_counts(di, g, plan, hashes + off, m, tl, false, s, cnt);
    for (uint32_t k = 0, pre = 0; e == cudaSuccess && k < plan.super_parts; pre += cnt[k], ++k)
      if (cnt[k])
        e = insert_chunk(di, blocks + plan.h_super_bounds[k] * 8, sub_geom(g, plan.h_super_bounds, k), plan.parts,
                         tl.keys + pre, cnt[k], sc, s);
  }
  free_scratch(sc, s);
  if (tl.keys) cudaFreeAsync(tl.keys, s);
  if (tl.counts) cudaFreeAsync(tl.counts, s);
  return e;
}

cudaError_t blocked_find(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                         const uint64_t* hashes, uint64_t n, void* out, bool bits, cudaStream_t s, bool dense_only) {
  if (n == 0) return cudaSuccess;
  const uint64_t cap = n < blocked_round() ? n : blocked_round();  // a multiple of 32 unless n is the whole batch
  CallScope scope(plan.ctx, s, scratch_bytes(cap, true));
  if (scope.error() != cudaSuccess) return scope.error();
  Scratch sc;
  TwoLevel tl;
  const bool two = plan.super_parts > 1;
  const bool whole = g.first == 0 && g.nb_local == g.nb_global;  // no key can fall outside the filter
  cudaError_t e = alloc_scratch(sc, cap, true, s, &scope);
  if (e == cudaSuccess && two) e = cudaMallocAsync(reinterpret_cast<void**>(&tl.keys), cap * sizeof(uint64_t), s);
  if (e == cudaSuccess && two) e = cudaMallocAsync(reinterpret_cast<void**>(&tl.pos), cap * sizeof(uint32_t), s);
  if (e == cudaSuccess && two) e = cudaMallocAsync(reinterpret_cast<void**>(&tl.ans), cap, s);
  if (e == cudaSuccess && two && bits) e = cudaMallocAsync(reinterpret_cast<void**>(&tl.bytes), cap, s);
  if (e == cudaSuccess && two)
    e = cudaMallocAsync(reinterpret_cast<void**>(&tl.counts), 2 * plan.super_parts * sizeof(uint64_t), s);
  std::vector<uint64_t> cnt;
  uint64_t start = 0;
  if (e == cudaSuccess && !two) {
    // the fused path sizes its own rounds over the whole batch
    e = try_find_fused(di, blocks, g, plan.parts, hashes, n, sc, cap, out, bits, s, whole, dense_only);
    if (e == cudaErrorNotSupported) e = cudaSuccess;
    else start = n;
  }
  for (uint64_t off = start; e == cudaSuccess && off < n; off += cap) {
    const uint64_t m = n - off < cap ? n - off : cap;
    void* dst = bits ? static_cast<void*>(static_cast<uint32_t*>(out) + off / 32)
                     : static_cast<void*>(static_cast<uint8_t*>(out) + off);
    if (!two) {
      e = find_chunk(di, blocks, g, plan.parts, hashes + off, m, sc, dst, bits, s, whole, dense_only);
      continue;
    }
    e = super_counts(di, g, plan, hashes + off, m, tl, true, s, cnt);
    for (uint32_t k = 0, pre = 0; e == cudaSuccess && k < plan.super_parts; pre += cnt[k], ++k)
      if (cnt[k])
        e = find_chunk(di, blocks + plan.h_super_bounds[k] * 8, sub_geom(g, plan.h_super_bounds, k), plan.parts,
                       tl.keys + pre, cnt[k], sc, tl.ans + pre, false, s, whole, dense_only);
    // grouped answers back to source order (then packed for bit output)
    uint8_t* bytes = bits ? tl.bytes : static_cast<uint8_t*>(dst);
    if (e == cudaSuccess && sbbf_scatter_u8(tl.ans, tl.pos, m, bytes, s) != SBBF_OK) e = cudaGetLastError();
    if (e == cudaSuccess && bits && sbbf_pack_bits(tl.bytes, m, static_cast<uint32_t*>(dst), s) != SBBF_OK)
      e = cudaGetLastError();
  }
  free_scratch(sc, s);
  if (tl.keys) cudaFreeAsync(tl.keys, s);
  if (tl.pos) cudaFreeAsync(tl.pos, s);
  if (tl.ans) cudaFreeAsync(tl.ans, s);
  if (tl.bytes) cudaFreeAsync(tl.bytes, s);
  if (tl.counts) cudaFreeAsync(tl.counts, s);
  return e;
}

// Keys given as several arrays (a rank's receive-window regions): each
// region's chunks take consecutive chunk slots of one scratch, so a single
// segment pass — one sweep of the filter through L2 — covers them all, with
// no staging copy. Single-level plans and batches up to blocked_round() keys;
// anything else returns cudaErrorNotSupported (the caller gathers instead).
namespace {
uint64_t region_chunks(const uint64_t* counts, uint32_t nr, std::vector<uint64_t>& off) {
  off.assign(nr + 1, 0);
  for (uint32_t r = 0; r < nr; ++r) off[r + 1] = off[r] + (counts[r] + kPartChunk - 1) / kPartChunk;
  return off[nr];
}
}  // namespace

cudaError_t blocked_insert_regions(const DeviceInfo& di, uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                                   const uint64_t* const* keys, const uint64_t* counts, uint32_t nr, cudaStream_t s) {
  std::vector<uint64_t> off;
  const uint64_t C = region_chunks(counts, nr, off);
  if (plan.super_parts > 1 || C * kPartChunk > blocked_round()) return cudaErrorNotSupported;
  if (C == 0) return cudaSuccess;
  Scratch sc;
  CallScope scope(plan.ctx, s, scratch_bytes(C * kPartChunk, false));
  if (scope.error() != cudaSuccess) return scope.error();
  cudaError_t e = alloc_scratch(sc, C * kPartChunk, false, s, &scope);
  for (uint32_t r = 0; e == cudaSuccess && r < nr; ++r)
    if (counts[r])
      e = chunk_partition(di, g, plan.parts, keys[r], counts[r], sc.keys + off[r] * kPartChunk, nullptr,
                          sc.boffs + off[r] * kBoffStride, s);
  if (e == cudaSuccess)
    e = launch_segments<true>(blocks, g, sc.keys, sc.boffs, plan.parts, C * kPartChunk, nullptr, s, sc.work, &di,
                              sc.flip);
  free_scratch(sc, s);
  return e;
}

cudaError_t blocked_find_regions(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                                 const uint64_t* const* keys, const uint64_t* counts, uint32_t nr, uint8_t* const* outs,
                                 cudaStream_t s, bool dense_only) {
  std::vector<uint64_t> off;
  const uint64_t C = region_chunks(counts, nr, off);
  if (plan.super_parts > 1 || C * kPartChunk > blocked_round()) return cudaErrorNotSupported;
  if (C == 0) return cudaSuccess;
  Scratch sc;
  uint8_t* bytes = nullptr;  // answers in the chunk layout: region r's at off[r] * kPartChunk
  CallScope scope(plan.ctx, s, scratch_bytes(C * kPartChunk, true));
  if (scope.error() != cudaSuccess) return scope.error();
  cudaError_t e = alloc_scratch(sc, C * kPartChunk, true, s, &scope);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&bytes), C * kPartChunk, s);
  // the fused sweep when the map packs and one launch takes every chunk
  // (routed keys can still include ones the shard does not own: sentinel map)
  BucketMap bm = make_map(g, plan.parts);
  FusedShape fs;
  uint64_t total = 0;
  for (uint32_t r = 0; r < nr; ++r) total += counts[r];
  const bool fused = e == cudaSuccess && find_fused() && !(dense_only && total < g.nb_local) &&
                     pack_map(bm, g.first == 0 && g.nb_local == g.nb_global) &&
                     fused_shape(di, bm, fs) == cudaSuccess && C <= fs.max_chunks();
  for (uint32_t r = 0; e == cudaSuccess && r < nr; ++r)
    if (counts[r])
      e = chunk_partition(di, g, plan.parts, keys[r], counts[r], sc.keys + off[r] * kPartChunk,
                          sc.pos16 + off[r] * kPartChunk, sc.boffs + off[r] * kBoffStride, s, fused ? &bm : nullptr);
  if (e == cudaSuccess && fused) {
    e = fused_sweep(fs, blocks, g, bm, sc, C, bytes, false, s);
  } else if (e == cudaSuccess) {
    e = launch_segments<false>(const_cast<uint32_t*>(blocks), g, sc.keys, sc.boffs, plan.parts, C * kPartChunk,
                               sc.ans, s, sc.work, &di, sc.flip);
    if (e == cudaSuccess) {
      note_launch();
      unpermute_kernel<<<static_cast<unsigned>(C), kUnpermThreads, 0, s>>>(sc.ans, sc.pos16, C * kPartChunk, bytes,
                                                                           false, sc.boffs);
      e = cudaGetLastError();
    }
  }
  for (uint32_t r = 0; e == cudaSuccess && r < nr; ++r)
    if (counts[r])
      e = cudaMemcpyAsync(outs[r], bytes + off[r] * kPartChunk, counts[r], cudaMemcpyDeviceToDevice, s);
  if (bytes) cudaFreeAsync(bytes, s);
  free_scratch(sc, s);
  return e;
}

}  // namespace sbbf

extern "C" int sbbf_bench_kernel_timing(int enable) {
  sbbf::KTimer& t = sbbf::ktimer();
  std::lock_guard<std::mutex> lock(t.mu);
  for (auto& p : t.pending) t.pool.emplace_back(std::get<1>(p), std::get<2>(p));
  t.pending.clear();
  for (int k = 0; k < sbbf::kKNum; ++k) {
    t.ms[k] = 0;
    t.n[k] = 0;
  }
  t.on.store(enable != 0, std::memory_order_relaxed);
  return SBBF_OK;
}

extern "C" int sbbf_bench_kernel_times(double* ms, uint64_t* launches, int n) {
  sbbf::KTimer& t = sbbf::ktimer();
  std::lock_guard<std::mutex> lock(t.mu);
  int rc = SBBF_OK;
  for (auto& p : t.pending) {
    float e = 0;
    const cudaEvent_t a = std::get<1>(p), b = std::get<2>(p);
    if (cudaEventSynchronize(b) == cudaSuccess && cudaEventElapsedTime(&e, a, b) == cudaSuccess) {
      t.ms[std::get<0>(p)] += e;
      t.n[std::get<0>(p)] += 1;
    } else {
      cudaGetLastError();
      rc = SBBF_ECUDA;
    }
    t.pool.emplace_back(a, b);
  }
  t.pending.clear();
  for (int k = 0; k < n && k < sbbf::kKNum; ++k) {
    if (ms) ms[k] = t.ms[k];
    if (launches) launches[k] = t.n[k];
  }
  return rc;
}
