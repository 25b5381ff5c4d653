// sbbf_blocked.cu — L2-blocked insert/lookup for filters larger than L2.
//
// A random 32-byte probe that misses L2 costs a full DRAM line fill
// (ncu: ~117 B of DRAM per key on a 1 GiB filter) and the HBM random-sector
// rate tops out at 37-43 G/s whatever the access path (LSU, TMA, gather4;
// profiles/r1_microbench_*.log). The blocked path trades that for streaming:
//
//   1. bucket the batch by filter slice (bucket_count + bucket_scatter:
//      8 B in, 8 B (+4 B source position) out per key),
//   2. process the grouped keys in slice order — CTAs are dispatched in
//      blockIdx order, so the keys in flight at any moment fall in one or two
//      slices (~16 MiB each) and their probes/atomics hit L2; every filter
//      line is fetched from HBM about once per chunk,
//   3. lookups set their answer bit at the key's source position with a red
//      into a chunk bitmap that stays L2-resident.
//
// Per-key HBM traffic ~ 8 (count) + 8 + 12 (scatter) + 12 (probe) +
// filter_bytes / chunk_keys, instead of a ~128-byte random line fill.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

constexpr uint64_t kBlockedChunk = uint64_t{1} << 28;  // keys per partition round (3.1 GB scratch)
constexpr int kProbeU = 8;
constexpr int kProbeThreads = 256;
constexpr uint64_t kProbeTile = kProbeThreads * kProbeU;

// ---------------------------------------------------------------------------
// bucket partition
// ---------------------------------------------------------------------------
// Bucket of a key = its local block scaled to [0, S) by a 32.32 fixed-point
// multiply: monotone in the block, so bucket k is a contiguous block range of
// ~nb/S blocks (neighbouring buckets may share a boundary block — harmless,
// each key is still handled on its own). S <= 64.
//
// Ranking inside a warp is a ballot "multisplit": for a BITS-bit bucket id,
// BITS ballots give every lane the mask of lanes holding its bucket (AND of
// ballot or ~ballot per bit). Per-warp running counts live in registers —
// lane l owns buckets l and l+32 — so there are no per-key shared-memory
// atomics (~2 cycles per lane on this part) and no __match_any_sync (which
// measured slower still: profiles/r1_blocked_partition.md).
constexpr int kPartThreads = 512;
constexpr int kPartWarps = kPartThreads / 32;
constexpr int kPartPerThread = 8;
constexpr uint64_t kPartChunk = kPartThreads * kPartPerThread;
constexpr int kMaxBuckets = 64;
constexpr int kMaxBits = 6;

struct BucketMap {
  uint64_t nb_global, first, nb_local, mult;  // mult = floor(S * 2^32 / nb_local)
  uint32_t S, bits;
  const uint64_t* bounds;  // optional exact bucket starts (local block ids), S entries
  bool top_bits;           // whole filter, S = 2^bits: bucket = top bits of the hash
};

__device__ __forceinline__ uint32_t bucket_of(uint64_t h, const BucketMap& bm) {
  // block_index is monotone in the hash, so the hash's top bits split the
  // filter into S contiguous block ranges without any 64-bit multiply
  if (bm.top_bits) return static_cast<uint32_t>(h >> (64 - bm.bits));
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

// Lanes whose bucket equals `v`, given the per-bit ballots of the warp.
template <int BITS>
__device__ __forceinline__ uint32_t lanes_with(uint32_t v, const uint32_t (&bal)[kMaxBits], uint32_t active) {
  uint32_t m = active;
#pragma unroll
  for (int k = 0; k < BITS; ++k) m &= ((v >> k) & 1u) ? bal[k] : ~bal[k];
  return m;
}

template <int BITS>
__device__ __forceinline__ void bit_ballots(uint32_t bk, uint32_t (&bal)[kMaxBits]) {
#pragma unroll
  for (int k = 0; k < BITS; ++k) bal[k] = __ballot_sync(0xffffffffu, (bk >> k) & 1u);
}

// One warp step over 32 keys: rank of each lane inside its bucket group and
// the per-bucket counts added to the lane-owned counters c0 (bucket = lane)
// and c1 (bucket = lane + 32).
template <int BITS>
__device__ __forceinline__ uint32_t warp_rank(uint32_t bk, bool valid, uint32_t lane, uint32_t& c0,
                                              uint32_t& c1) {
  const uint32_t active = __ballot_sync(0xffffffffu, valid);
  uint32_t bal[kMaxBits];
  bit_ballots<BITS>(bk, bal);
  const uint32_t peers = lanes_with<BITS>(bk, bal, active);
  // prior count of my bucket in this warp, from the lane that owns it
  uint32_t prior = __shfl_sync(0xffffffffu, c0, bk & 31);
  if constexpr (BITS > 5) {
    const uint32_t p1 = __shfl_sync(0xffffffffu, c1, bk & 31);
    prior = (bk & 32) ? p1 : prior;
    c1 += __popc(lanes_with<BITS>(lane + 32, bal, active));
  }
  c0 += __popc(lanes_with<BITS>(lane, bal, active));
  return prior + __popc(peers & ((1u << lane) - 1u));
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

template <int BITS>
__global__ void __launch_bounds__(kPartThreads, 2) bucket_count_kernel(const uint64_t* __restrict__ hashes,
                                                                       uint64_t n, BucketMap bm,
                                                                       uint32_t* __restrict__ cta_hist) {
  __shared__ unsigned int cta[kMaxBuckets];
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t pol = dev::policy_evict_first();
  if (threadIdx.x < kMaxBuckets) cta[threadIdx.x] = 0;
  uint32_t c0 = 0, c1 = 0;
  uint64_t ch0, ch1;
  cta_chunk_range(n, ch0, ch1);
  // Software pipeline: the next chunk's loads are in flight while this
  // chunk's ballots run (the kernel is otherwise latency bound).
  uint64_t nxt[kPartPerThread];
#pragma unroll
  for (int j = 0; j < kPartPerThread; ++j) {
    const uint64_t i = ch0 * kPartChunk + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
    nxt[j] = (ch0 < ch1 && i < n) ? dev::ld_stream_u64(hashes + i, pol) : 0;
  }
  for (uint64_t ch = ch0; ch < ch1; ++ch) {
    const uint64_t base = ch * kPartChunk;
    uint64_t h[kPartPerThread];
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      h[j] = nxt[j];
      const uint64_t i = base + kPartChunk + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
      nxt[j] = (ch + 1 < ch1 && i < n) ? dev::ld_stream_u64(hashes + i, pol) : 0;
    }
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
      const uint32_t bk = i < n ? bucket_of(h[j], bm) : 0u;
      const uint32_t active = __ballot_sync(0xffffffffu, i < n);
      uint32_t bal[kMaxBits];
      bit_ballots<BITS>(bk, bal);
      c0 += __popc(lanes_with<BITS>(lane, bal, active));
      if constexpr (BITS > 5) c1 += __popc(lanes_with<BITS>(lane + 32, bal, active));
    }
  }
  __syncthreads();
  if (lane < bm.S && c0) atomicAdd(&cta[lane], c0);
  if (lane + 32 < bm.S && c1) atomicAdd(&cta[lane + 32], c1);
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

template <int BITS>
__global__ void __launch_bounds__(kPartThreads, 2) bucket_scatter_kernel(
    const uint64_t* __restrict__ hashes, uint64_t n, BucketMap bm,
    const unsigned long long* __restrict__ cta_base, uint64_t* __restrict__ out, uint32_t* __restrict__ pos,
    RouteOut route = RouteOut{}, const unsigned long long* __restrict__ counts = nullptr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScatterSmem& sm = *reinterpret_cast<ScatterSmem*>(smem_raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
      h[j] = i < n ? dev::ld_stream_u64(hashes + i, pol) : 0;
    }
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x;
      const bool valid = i < n;
      bk[j] = valid ? bucket_of(h[j], bm) : 0u;
      off[j] = warp_rank<BITS>(bk[j], valid, lane, c0, c1);
      if (!valid) bk[j] = 0xffffffffu;
    }
    sm.wcnt[warp][lane] = c0;
    sm.wcnt[warp][lane + 32] = c1;
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
#pragma unroll
    for (int j = 0; j < kPartPerThread; ++j) {
      if (bk[j] != 0xffffffffu) {
        const uint32_t loc = sm.boff[bk[j]] + sm.wcnt[warp][bk[j]] + off[j];
        sm.key[loc] = h[j];
        sm.pos[loc] = static_cast<uint32_t>(base + static_cast<uint64_t>(j) * kPartThreads + threadIdx.x);
        sm.bk[loc] = static_cast<uint8_t>(bk[j]);
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += kPartThreads) {
      const uint32_t b = sm.bk[i];
      const uint64_t slot = sm.gbase[b] + (i - sm.boff[b]);
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

template <int BITS>
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
      bucket_scatter_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      static_cast<int>(sizeof(ScatterSmem)));
  if (e == cudaSuccess) e = attr;
  if (e == cudaSuccess) {
    note_launch();
    bucket_count_kernel<BITS><<<static_cast<unsigned>(grid), kPartThreads, 0, s>>>(hashes, m, bm, hist);
    note_launch();
    bucket_scan_kernel<<<1, kMaxBuckets, 0, s>>>(hist, static_cast<uint32_t>(grid), bm.S,
                                                 reinterpret_cast<unsigned long long*>(d_counts), bases);
    note_launch();
    bucket_scatter_kernel<BITS><<<static_cast<unsigned>(grid), kPartThreads, sizeof(ScatterSmem), s>>>(
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
  const uint64_t grid = m ? grid_for(m, kPartChunk, di.sms, 2) : 1;
  switch (bm.bits) {
    case 1: return bucket_partition_bits<1>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    case 2: return bucket_partition_bits<2>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    case 3: return bucket_partition_bits<3>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    case 4: return bucket_partition_bits<4>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    case 5: return bucket_partition_bits<5>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    case 6: return bucket_partition_bits<6>(grid, bm, hashes, m, d_counts, d_out, d_pos, s, route);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// grouped probe
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kProbeThreads, 2) probe_grouped_kernel(
    const uint32_t* __restrict__ blocks, Geom g, const uint64_t* __restrict__ keys,
    const uint32_t* __restrict__ pos, uint64_t m, uint32_t* __restrict__ bitmap) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kProbeTile + threadIdx.x;
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t keep = dev::policy_evict_last();
  uint64_t h[kProbeU];
  uint32_t p[kProbeU];
#pragma unroll
  for (int u = 0; u < kProbeU; ++u) {
    const uint64_t i = base + static_cast<uint64_t>(u) * kProbeThreads;
    h[u] = i < m ? dev::ld_stream_u64(keys + i, pol) : 0;
    p[u] = i < m ? dev::ld_stream_u32(pos + i, pol) : 0;
  }
  dev::Block8 b[kProbeU];
  uint32_t ok_mask = 0;
#pragma unroll
  for (int u = 0; u < kProbeU; ++u) {
    const uint64_t blk = dev::block_index(h[u], g.nb_global) - g.first;
    const bool ok = blk < g.nb_local;
    ok_mask |= static_cast<uint32_t>(ok) << u;
    dev::ld_block_nc_normal(blocks + (ok ? blk : 0) * 8, b[u]);
  }
#pragma unroll
  for (int u = 0; u < kProbeU; ++u) {
    const uint64_t i = base + static_cast<uint64_t>(u) * kProbeThreads;
    if (i < m && ((ok_mask >> u) & 1u) && dev::block_contains(b[u], h[u]))
      dev::red_or(bitmap + (p[u] >> 5), 1u << (p[u] & 31), keep);  // chunk bitmap stays in L2
  }
}

__global__ void expand_bits_kernel(const uint32_t* __restrict__ bits, uint64_t n, uint8_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<uint8_t>((bits[i >> 5] >> (i & 31)) & 1u);
}

struct Scratch {
  uint64_t* keys = nullptr;
  uint32_t* pos = nullptr;
  uint64_t* counts = nullptr;  // [2][S]: counts, cursor
  uint32_t* bits = nullptr;
};

cudaError_t alloc_scratch(Scratch& sc, uint64_t cap, uint32_t parts, bool with_pos, bool with_bits,
                          cudaStream_t s) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sc.keys), cap * sizeof(uint64_t), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&sc.counts), 2 * parts * sizeof(uint64_t), s);
  if (e == cudaSuccess && with_pos) e = cudaMallocAsync(reinterpret_cast<void**>(&sc.pos), cap * sizeof(uint32_t), s);
  if (e == cudaSuccess && with_bits)
    e = cudaMallocAsync(reinterpret_cast<void**>(&sc.bits), ((cap + 31) / 32) * sizeof(uint32_t), s);
  return e;
}

void free_scratch(Scratch& sc, cudaStream_t s) {
  if (sc.keys) cudaFreeAsync(sc.keys, s);
  if (sc.pos) cudaFreeAsync(sc.pos, s);
  if (sc.counts) cudaFreeAsync(sc.counts, s);
  if (sc.bits) cudaFreeAsync(sc.bits, s);
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

cudaError_t blocked_insert(const DeviceInfo& di, uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                           const uint64_t* hashes, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t cap = n < kBlockedChunk ? n : kBlockedChunk;
  Scratch sc;
  cudaError_t e = alloc_scratch(sc, cap, plan.parts, false, false, s);
  for (uint64_t off = 0; e == cudaSuccess && off < n; off += cap) {
    const uint64_t m = n - off < cap ? n - off : cap;
    e = bucket_partition(di, g, plan.parts, hashes + off, m, sc.counts, sc.counts + plan.parts, sc.keys,
                         nullptr, s);
    // test-before-set: grouped duplicates (config 4's hot keys arrive back to
    // back) skip the atomic once their bits are in.
    if (e == cudaSuccess) e = launch_insert_ordered(di, blocks, g, sc.keys, m, /*test=*/true, s);
  }
  free_scratch(sc, s);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t blocked_find(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                         const uint64_t* hashes, uint64_t n, void* out, bool bits, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t cap = n < kBlockedChunk ? n : kBlockedChunk;  // a multiple of 32 unless n is the whole batch
  Scratch sc;
  cudaError_t e = alloc_scratch(sc, cap, plan.parts, true, !bits, s);
  for (uint64_t off = 0; e == cudaSuccess && off < n; off += cap) {
    const uint64_t m = n - off < cap ? n - off : cap;
    uint32_t* bm = bits ? static_cast<uint32_t*>(out) + off / 32 : sc.bits;
    e = cudaMemsetAsync(bm, 0, ((m + 31) / 32) * sizeof(uint32_t), s);
    if (e == cudaSuccess)
      e = bucket_partition(di, g, plan.parts, hashes + off, m, sc.counts, sc.counts + plan.parts, sc.keys,
                           sc.pos, s);
    if (e != cudaSuccess) break;
    note_launch();
    probe_grouped_kernel<<<static_cast<unsigned>((m + kProbeTile - 1) / kProbeTile), kProbeThreads, 0, s>>>(
        blocks, g, sc.keys, sc.pos, m, bm);
    e = cudaGetLastError();
    if (e == cudaSuccess && !bits) {
      note_launch();
      expand_bits_kernel<<<static_cast<unsigned>(grid_for(m, 1024, di.sms, 8)), 256, 0, s>>>(
          bm, m, static_cast<uint8_t*>(out) + off);
      e = cudaGetLastError();
    }
  }
  free_scratch(sc, s);
  return e;
}

}  // namespace sbbf
