// sbbf_kernels.cu — hand-written sm_100a kernels for batched SBBF insert/lookup.
//
// Reference hot loops being replaced (paths relative to /root/reference/proj/):
//   add_many_avx2  core/src/filter.cpp:79-84   (per key: load 32 B, OR mask, store)
//   find_many_avx2 core/src/filter.cpp:86-93   (per key: load 32 B, vptest, 1 byte out)
//
// Design (DESIGN.md §3 has the roofline for each):
//   * insert_wide     — 4 threads per key, one `red.global.or.b64` per lane pair.
//     The L2 atomic unit is op-bound, so 4 ops/key beat 8 (insert_lane8) and
//     32 scattered ops/warp-instruction (insert_thread). Atomic OR is exact:
//     OR is commutative/associative/idempotent, so any interleaving yields the
//     reference's bytes.
//   * insert_*_test   — load first, red only lanes whose bits are missing (bits
//     are monotone): a miss is filled by the faster read path and
//     duplicate/hot keys (config 4's Zipf) skip the atomic.
//   * find_pipe       — one thread per key, U = 4 keys in flight per thread plus
//     the next tile's hashes (software pipelined), one 256-bit LDG per key
//     (LDG.E.256), hashes streamed evict-first, results either 0/1 bytes
//     (drop-in) or a __ballot_sync-packed bitmap; launched as a programmatic
//     dependent of a preceding insert; kKeys hashes u64 keys (XXH64) as they
//     stream in.
//   * find_smem       — small filters (<= ~200 KiB, e.g. config 1) are staged
//     into shared memory per CTA with cp.async.bulk (TMA bulk copy, mbarrier
//     completion) and probed with two 128-bit LDS per key.
//
// Every kernel takes a Geom: the block index is computed against the GLOBAL
// bucket count and offset by the shard's first block, so a shard of a
// multi-GPU filter (sharded.py) keeps the reference's block_index exactly.
// Keys outside [first, first + nb_local) are ignored by inserts and answer 0
// in lookups (the router never sends them).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

using dev::Block8;

constexpr int kThreads = 256;

// Local block of `h` and whether this shard owns it.
__device__ __forceinline__ uint64_t local_block(uint64_t h, const Geom& g, bool& ok) {
  const uint64_t b = dev::block_index(h, g.nb_global) - g.first;
  ok = b < g.nb_local;
  return ok ? b : 0;
}

// ---------------------------------------------------------------------------
// insert
// ---------------------------------------------------------------------------
// __launch_bounds__ minimum-blocks hints below are load-bearing: without them
// ptxas minimises registers by sinking each load next to its use, which
// serialises the independent sector accesses (checked in SASS).
template <bool kTest>
__global__ void __launch_bounds__(kThreads, 4) insert_lane8_kernel(uint32_t* __restrict__ blocks, Geom g,
                                                                   const uint64_t* __restrict__ hashes,
                                                                   uint64_t n) {
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 3;  // which of the 4 keys of a round
  const int word = lane & 7;  // which lane of the block this thread owns
  const uint32_t seed = dev::lane_seed_rt(word);
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t keep = dev::policy_evict_last();
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint64_t ntiles = (n + 31) >> 5;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t base = t << 5;
    const uint64_t idx = base + lane;
    const uint64_t h = idx < n ? dev::ld_stream_u64(hashes + idx, pol) : 0;
    const uint32_t valid = __ballot_sync(0xffffffffu, idx < n);
    uint32_t* ptr[8];
    uint32_t bit[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int k = r * 4 + sub;
      const uint64_t hk = __shfl_sync(0xffffffffu, h, k);
      bool ok;
      ptr[r] = blocks + local_block(hk, g, ok) * 8 + word;
      bit[r] = (((valid >> k) & 1u) && ok) ? dev::lane_bit(static_cast<uint32_t>(hk), seed) : 0u;
    }
    if constexpr (kTest) {
      uint32_t cur[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) cur[r] = bit[r] ? dev::ld_lane(ptr[r], keep) : ~0u;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (bit[r] & ~cur[r]) dev::red_or(ptr[r], bit[r], keep);
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (bit[r]) dev::red_or(ptr[r], bit[r], keep);
    }
  }
}

// 4 threads per key, one 64-bit `red.global.or.b64` per lane pair: half the
// L2 atomic operations of insert_lane8 (120 vs 85 G keys/s on an L2-resident
// buffer, scripts/microbench.cu). Lane 2w is the low half of u64 word w
// (little-endian lanes, filter.hpp:23-24).
// kKeys: the input is u64 keys, hashed on the fly with XXH64(seed) (the
// reference's kHasherXxh64 frontend fused into the insert).
// kHint: reds carry an L2 evict-last policy (filters near or beyond L2 size);
// without it an L2-resident filter's 1M-key insert is 1.2 us faster
// (scripts/microbench_red.cu: 15.2 vs 16.4 us).
// kSplit: this pass inserts only the keys whose top hash bits (h >> psh)
// equal pid — one contiguous block range of a whole filter (block_index is
// monotone in the hash) — so a filter somewhat larger than L2 is inserted
// range by range, each range L2-resident while its reds land.
template <bool kTest, bool kKeys = false, int kT = 4, bool kHint = true, bool kSplit = false>
__global__ void __launch_bounds__(kThreads, 4) insert_wide_kernel(uint32_t* __restrict__ blocks, Geom g,
                                                                  const uint64_t* __restrict__ hashes,
                                                                  uint64_t n, uint64_t seed = 0, uint32_t psh = 63,
                                                                  uint64_t pid = 0) {
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 2;   // which of the 8 keys of a round
  const int pair = lane & 3;   // which 64-bit lane pair of the block this thread owns
  const uint32_t seed_lo = dev::lane_seed_rt(2 * pair), seed_hi = dev::lane_seed_rt(2 * pair + 1);
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t keep = dev::policy_evict_last();
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  // A warp step covers kT tiles of 32 keys: the kT hash loads are issued
  // together so one DRAM round trip feeds 4*kT atomic rounds.
  const uint64_t nsteps = (n + 32 * kT - 1) / (32 * kT);
  // Programmatic dependent launch: let a following lookup grid get scheduled
  // now (it waits in griddepcontrol.wait for this grid to finish before it
  // reads the filter) so its launch latency hides behind this kernel's tail.
  asm volatile("griddepcontrol.launch_dependents;");
  if constexpr (kSplit) {
    // compact this pass's keys per warp in shared memory, then run the
    // 4-lanes-per-key red rounds over them only
    __shared__ uint64_t cbuf[kThreads / 32][32 * kT];
    uint64_t* cb = cbuf[threadIdx.x >> 5];
    for (uint64_t t = warp; t < nsteps; t += nwarps) {
      const uint64_t base = t * (32 * kT);
      uint64_t h[kT];
#pragma unroll
      for (int j = 0; j < kT; ++j) {
        const uint64_t idx = base + j * 32 + lane;
        h[j] = idx < n ? dev::to_hash<kKeys>(dev::ld_stream_u64(hashes + idx, pol), seed) : 0;
      }
      uint32_t total = 0;
#pragma unroll
      for (int j = 0; j < kT; ++j) {
        const bool in = base + j * 32 + lane < n && (h[j] >> psh) == pid;
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        if (in) cb[total + __popc(bal & ((1u << lane) - 1u))] = h[j];
        total += __popc(bal);
      }
      __syncwarp();
      for (uint32_t k0 = 0; k0 < total; k0 += 8) {
        const uint32_t k = k0 + sub;
        if (k < total) {
          const uint64_t hk = cb[k];
          const uint32_t low = static_cast<uint32_t>(hk);
          bool ok;
          uint64_t* ptr = reinterpret_cast<uint64_t*>(blocks + local_block(hk, g, ok) * 8) + pair;
          const uint64_t mask = (static_cast<uint64_t>(dev::lane_bit(low, seed_hi)) << 32) | dev::lane_bit(low, seed_lo);
          if (ok) {
            if constexpr (kHint) dev::red_or64(ptr, mask, keep);
            else dev::red_or64_nohint(ptr, mask);
          }
        }
      }
      __syncwarp();
    }
    return;
  }
  for (uint64_t t = warp; t < nsteps; t += nwarps) {
    const uint64_t base = t * (32 * kT);
    uint64_t h[kT];
#pragma unroll
    for (int j = 0; j < kT; ++j) {
      const uint64_t idx = base + j * 32 + lane;
      h[j] = idx < n ? dev::to_hash<kKeys>(dev::ld_stream_u64(hashes + idx, pol), seed) : 0;
    }
#pragma unroll
    for (int j = 0; j < kT; ++j) {
      const uint32_t valid = __ballot_sync(0xffffffffu, base + j * 32 + lane < n);
      if (valid == 0) break;
      uint64_t* ptr[4];
      uint64_t mask[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int k = r * 8 + sub;
        const uint64_t hk = __shfl_sync(0xffffffffu, h[j], k);
        const uint32_t low = static_cast<uint32_t>(hk);
        bool ok;
        ptr[r] = reinterpret_cast<uint64_t*>(blocks + local_block(hk, g, ok) * 8) + pair;
        mask[r] = (((valid >> k) & 1u) && ok)
                      ? (static_cast<uint64_t>(dev::lane_bit(low, seed_hi)) << 32) | dev::lane_bit(low, seed_lo)
                      : 0ull;
      }
      if constexpr (kTest) {
        uint64_t cur[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) cur[r] = mask[r] ? dev::ld_pair(ptr[r], keep) : ~0ull;
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (mask[r] & ~cur[r]) dev::red_or64(ptr[r], mask[r], keep);
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (!mask[r]) continue;
          if constexpr (kHint) dev::red_or64(ptr[r], mask[r], keep);
          else dev::red_or64_nohint(ptr[r], mask[r]);
        }
      }
    }
  }
}

// Baseline variant: one thread per key, eight word atomics per key.
__global__ void __launch_bounds__(kThreads) insert_thread_kernel(uint32_t* __restrict__ blocks, Geom g,
                                                                 const uint64_t* __restrict__ hashes,
                                                                 uint64_t n) {
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t keep = dev::policy_evict_last();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    const uint64_t h = dev::ld_stream_u64(hashes + i, pol);
    bool ok;
    uint32_t* b = blocks + local_block(h, g, ok) * 8;
    if (!ok) continue;
    const uint32_t low = static_cast<uint32_t>(h);
#pragma unroll
    for (int w = 0; w < 8; ++w) dev::red_or(b + w, dev::lane_bit(low, dev::lane_seed(w)), keep);
  }
}

// ---------------------------------------------------------------------------
// lookup from L2/HBM
// ---------------------------------------------------------------------------
// Warp tile = 32*U consecutive keys; lane l owns keys base + u*32 + l. All U
// hash loads, then all U block loads are issued before any is consumed, so
// each thread keeps U independent 32-byte sector reads in flight.
// Software-pipelined variant: the next tile's hashes are loaded while this
// tile's block loads are in flight, so the HBM latency of the hash stream is
// off the per-warp critical path.
template <int U, bool kBits, int kMinBlocks = 2, bool kKeys = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    find_pipe_kernel(const uint32_t* __restrict__ blocks, Geom g, const uint64_t* __restrict__ hashes,
                     uint64_t n, void* __restrict__ out, uint64_t seed = 0) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  constexpr uint64_t kTile = 32 * U;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  // hn holds the next tile's raw inputs; with kKeys the XXH64 is applied when
  // the tile is consumed, so the prefetch never waits on its own loads
  // Every global read, the caller's hashes included, comes after
  // griddepcontrol.wait: the previous grid on the stream may be the one that
  // produced the hashes (a key-hashing or generator kernel), and its writes
  // are only guaranteed visible past the wait. The early launch still hides
  // this grid's launch and CTA rasterisation behind the previous grid's tail.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint64_t hn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t idx = warp * kTile + u * 32 + lane;
    hn[u] = (warp < ntiles && idx < n) ? dev::ld_stream_u64(hashes + idx, pol) : 0;
  }
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t base = t * kTile;
    uint64_t h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) h[u] = dev::to_hash<kKeys>(hn[u], seed);
    Block8 b[U];
    uint32_t owned = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool ok;
      dev::ld_block_nc(blocks + local_block(h[u], g, ok) * 8, b[u]);
      owned |= static_cast<uint32_t>(ok) << u;
    }
    const uint64_t tn = t + nwarps;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = tn * kTile + u * 32 + lane;
      hn[u] = (tn < ntiles && idx < n) ? dev::ld_stream_u64(hashes + idx, pol) : 0;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = base + u * 32 + lane;
      const bool hit = dev::block_contains(b[u], h[u]) && ((owned >> u) & 1u) && idx < n;
      if constexpr (kBits) {
        const uint32_t word = __ballot_sync(0xffffffffu, hit);
        if (lane == u) mine = word;
      } else {
        if (idx < n) dev::st_stream_u8(static_cast<uint8_t*>(out) + idx, hit ? 1u : 0u);
      }
    }
    if constexpr (kBits) {
      const uint64_t nwords = (n + 31) >> 5;
      const uint64_t widx = (base >> 5) + lane;
      if (lane < U && widx < nwords) dev::st_stream_u32(static_cast<uint32_t*>(out) + widx, mine);
    }
  }
}

// ---------------------------------------------------------------------------
// lookup from shared memory (small filters)
// ---------------------------------------------------------------------------
// Whole-filter lookup (the single-GPU case: no shard offset, no ownership
// test), register-lean: after a block's address is formed only the low 32
// hash bits stay live (60-69 registers against find_pipe's 78). The next
// tile's hashes load while this tile's sectors are in flight, as in
// find_pipe. Config 2: 190.2 vs 188.5 Gkeys/s per step (profiles/r1_find_tuning.md).
// kSplit: one pass of a range-split lookup over a filter somewhat larger than
// L2 — only keys whose top hash bits (h >> psh) equal pid are probed, so this
// pass's probes stay in one L2-resident block range; the first pass stores
// the bitmap words, later passes OR theirs in (bytes: each pass stores its
// own keys' bytes).
template <int U, bool kBits, int kMinBlocks, bool kKeys = false, bool kSplit = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    find_whole_kernel(const uint32_t* __restrict__ blocks, uint64_t nb, const uint64_t* __restrict__ hashes,
                      uint64_t n, void* __restrict__ out, uint64_t seed = 0, uint32_t psh = 63, uint64_t pid = 0,
                      bool first = true) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  constexpr uint64_t kTile = 32 * U;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  // Every global read, the caller's hashes included, comes after
  // griddepcontrol.wait: the previous grid on the stream may be the one that
  // produced the hashes (a key-hashing or generator kernel), and its writes
  // are only guaranteed visible past the wait. The early launch still hides
  // this grid's launch and CTA rasterisation behind the previous grid's tail.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint64_t hn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t idx = warp * kTile + u * 32 + lane;
    hn[u] = (warp < ntiles && idx < n) ? dev::ld_stream_u64(hashes + idx, pol) : 0;
  }
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t base = t * kTile;
    uint32_t lo[U];
    Block8 b[U];
    uint32_t mine_part = 0;  // kSplit: bit u = key u of this lane is in this pass's range
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t h = dev::to_hash<kKeys>(hn[u], seed);  // XXH64 at consumption (kKeys)
      lo[u] = static_cast<uint32_t>(h);
      SBBF_DCHECK(dev::block_index(h, nb) < nb);
      if constexpr (kSplit) {
        const bool in = (h >> psh) == pid;
        mine_part |= static_cast<uint32_t>(in) << u;
        if (in) dev::ld_block_nc(blocks + dev::block_index(h, nb) * 8, b[u]);
      } else {
        dev::ld_block_nc(blocks + dev::block_index(h, nb) * 8, b[u]);
      }
    }
    const uint64_t tn = t + nwarps;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = tn * kTile + u * 32 + lane;
      hn[u] = (tn < ntiles && idx < n) ? dev::ld_stream_u64(hashes + idx, pol) : 0;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = base + u * 32 + lane;
      uint32_t missing = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) missing |= dev::lane_bit(lo[u], dev::lane_seed(i)) & ~b[u].w[i];
      const bool in = !kSplit || ((mine_part >> u) & 1u);
      const bool hit = missing == 0 && idx < n && in;
      if constexpr (kBits) {
        const uint32_t word = __ballot_sync(0xffffffffu, hit);
        if (lane == u) mine = word;
      } else {
        if (idx < n && in) dev::st_stream_u8(static_cast<uint8_t*>(out) + idx, hit ? 1u : 0u);
      }
    }
    if constexpr (kBits) {
      const uint64_t nwords = (n + 31) >> 5;
      const uint64_t widx = (base >> 5) + lane;
      if (lane < U && widx < nwords) {
        // range-split passes: the bitmap stays evict-first in L2 (it would
        // otherwise push the probed half of the filter out between passes)
        if (!kSplit) dev::st_stream_u32(static_cast<uint32_t*>(out) + widx, mine);
        else if (first) dev::st_stream_u32_ef(static_cast<uint32_t*>(out) + widx, mine, pol);
        else if (mine) dev::red_or(static_cast<uint32_t*>(out) + widx, mine, pol);
      }
    }
  }
}

// One range-split lookup pass, compacted (bitmap output): each warp takes
// 256 consecutive keys, moves this pass's keys (top 32 hash bits in
// [lo, lo + span): block_index is monotone in the hash, so that is one
// contiguous block range) to
// the front of a per-warp shared buffer with their in-tile index, probes
// only those (full warps, up to 4 sector loads in flight per lane), and
// assembles the 8 bitmap words of the 256 keys in shared memory. The first
// pass stores the words, later passes OR theirs in.
template <int kPU = 4, int kMinSB = 3, int kSplitTile = 256>
__global__ void __launch_bounds__(kThreads, kMinSB)
    find_split_kernel(const uint32_t* __restrict__ blocks, uint64_t nb, const uint64_t* __restrict__ hashes,
                      uint64_t n, uint32_t* __restrict__ out, uint64_t lo, uint64_t span, bool first) {
  __shared__ uint64_t ckey[kThreads / 32][kSplitTile];
  __shared__ uint8_t cidx[kThreads / 32][kSplitTile];
  __shared__ uint32_t cbits[kThreads / 32][kSplitTile / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint64_t ntiles = (n + kSplitTile - 1) / kSplitTile;
  const uint64_t nwords = (n + 31) >> 5;
  if (lane < kSplitTile / 32) cbits[w][lane] = 0;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // filter / bitmap only after the previous grid
  // (a register prefetch of the next tile's hashes measured slower: 107
  // registers, 2 CTAs/SM, 131.1 vs 148.2 Gkeys/s on config 3)
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t base = t * kSplitTile;
    uint64_t h[kSplitTile / 32];
#pragma unroll
    for (int k = 0; k < kSplitTile / 32; ++k) {
      const uint64_t idx = base + k * 32 + lane;
      h[k] = idx < n ? dev::ld_stream_u64(hashes + idx, pol) : 0;
    }
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < kSplitTile / 32; ++k) {
      const bool in = base + k * 32 + lane < n && (h[k] >> 32) - lo < span;
      const uint32_t bal = __ballot_sync(0xffffffffu, in);
      if (in) {
        const uint32_t pos = total + __popc(bal & ((1u << lane) - 1u));
        ckey[w][pos] = h[k];
        cidx[w][pos] = static_cast<uint8_t>(k * 32 + lane);
      }
      total += __popc(bal);
    }
    __syncwarp();
    for (uint32_t r0 = 0; r0 < total; r0 += 32 * kPU) {
      Block8 b[kPU];
      uint64_t hk[kPU];
#pragma unroll
      for (int u = 0; u < kPU; ++u) {
        const uint32_t j = r0 + u * 32 + lane;
        hk[u] = j < total ? ckey[w][j] : 0;
        if (j < total) dev::ld_block_nc(blocks + dev::block_index(hk[u], nb) * 8, b[u]);
      }
#pragma unroll
      for (int u = 0; u < kPU; ++u) {
        const uint32_t j = r0 + u * 32 + lane;
        if (j < total && dev::block_contains(b[u], hk[u])) {
          const uint32_t ci = cidx[w][j];
          atomicOr(&cbits[w][ci >> 5], 1u << (ci & 31));
        }
      }
    }
    __syncwarp();
    if (lane < kSplitTile / 32) {
      const uint64_t widx = (base >> 5) + lane;
      const uint32_t word = cbits[w][lane];
      cbits[w][lane] = 0;
      if (widx < nwords) {
        // evict-first in L2: the bitmap must not displace the probed half
        if (first) dev::st_stream_u32_ef(out + widx, word, pol);
        else if (word) dev::red_or(out + widx, word, pol);
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <bool kBits>
__global__ void __launch_bounds__(1024, 1) find_smem_kernel(const uint32_t* __restrict__ blocks, Geom g,
                                                            const uint64_t* __restrict__ hashes,
                                                            uint64_t n, void* __restrict__ out) {
  extern __shared__ __align__(128) uint4 sfilter[];
  __shared__ __align__(8) uint64_t mbar;
  const uint32_t bytes = static_cast<uint32_t>(g.nb_local * 32);
  const uint32_t bar = smem_u32(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    constexpr uint32_t kChunk = 16384;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t sz = bytes - off < kChunk ? bytes - off : kChunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(reinterpret_cast<const char*>(sfilter) + off)),
          "l"(reinterpret_cast<const char*>(blocks) + off), "r"(sz), "r"(bar)
          : "memory");
    }
  }
  // Wait for the bulk copy (phase 0).
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar)
          : "memory");
    }
  }

  const int lane = threadIdx.x & 31;
  const uint64_t pol = dev::policy_evict_first();
  constexpr int U = 4;
  constexpr uint64_t kTile = 32 * U;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t base = t * kTile;
    uint64_t h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = base + u * 32 + lane;
      h[u] = idx < n ? dev::ld_stream_u64(hashes + idx, pol) : 0;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = base + u * 32 + lane;
      bool ok;
      const uint4* p = sfilter + local_block(h[u], g, ok) * 2;
      const uint4 lo = p[0], hi = p[1];
      Block8 b{{lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w}};
      const bool hit = dev::block_contains(b, h[u]) && ok && idx < n;
      if constexpr (kBits) {
        const uint32_t word = __ballot_sync(0xffffffffu, hit);
        if (lane == u) mine = word;
      } else {
        if (idx < n) dev::st_stream_u8(static_cast<uint8_t*>(out) + idx, hit ? 1u : 0u);
      }
    }
    if constexpr (kBits) {
      const uint64_t nwords = (n + 31) >> 5;
      const uint64_t widx = (base >> 5) + lane;
      if (lane < U && widx < nwords) dev::st_stream_u32(static_cast<uint32_t*>(out) + widx, mine);
    }
  }
}

// ---------------------------------------------------------------------------
// free functions (known-answer tests)
// ---------------------------------------------------------------------------
__global__ void block_index_kernel(const uint64_t* __restrict__ h, uint64_t n, uint64_t nb,
                                   uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = dev::block_index(h[i], nb);
}

__global__ void make_mask_kernel(const uint64_t* __restrict__ h, uint64_t n,
                                 uint32_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t low = static_cast<uint32_t>(h[i]);
#pragma unroll
    for (int w = 0; w < 8; ++w) out[i * 8 + w] = dev::lane_bit(low, dev::lane_seed(w));
  }
}

// XXH64 of u64 keys (hash_u64_key, hash.cpp:108-114) and of byte strings
// (hash_key, hash.cpp:100-106; key i = data[offsets[i], offsets[i+1])).
__global__ void hash_u64_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint64_t seed,
                                uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = dev::xxh64_u64(keys[i], seed);
}

__global__ void hash_bytes_kernel(const uint8_t* __restrict__ data, const uint64_t* __restrict__ offsets,
                                  uint64_t n, uint64_t seed, uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t b = offsets[i], e = offsets[i + 1];
    out[i] = dev::xxh64_bytes(data + b, e - b, seed);
  }
}

// hash_key(std::to_string(counter), seed) for counters start .. start+n-1:
// the reference's KeyMode::kByteStrings keys (tools/harness.cpp:60-65),
// decimal digits built in registers, then XXH64 over them.
__global__ void hash_decimal_kernel(uint64_t start, uint64_t n, uint64_t seed, uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t c = start + i;
    uint8_t rev[20], buf[24];
    int len = 0;
    do {
      rev[len++] = static_cast<uint8_t>('0' + c % 10);
      c /= 10;
    } while (c);
    for (int k = 0; k < len; ++k) buf[k] = rev[len - 1 - k];
    out[i] = dev::xxh64_bytes(buf, static_cast<uint64_t>(len), seed);
  }
}

std::atomic<uint64_t> g_launches{0};

}  // namespace

cudaError_t launch_hash_u64(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  hash_u64_kernel<<<static_cast<unsigned>(grid_for(n, 1024, 148, 16)), 256, 0, s>>>(keys, n, seed, out);
  return cudaGetLastError();
}

cudaError_t launch_hash_bytes(const uint8_t* data, const uint64_t* offsets, uint64_t n, uint64_t seed,
                              uint64_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  hash_bytes_kernel<<<static_cast<unsigned>(grid_for(n, 256, 148, 16)), 128, 0, s>>>(data, offsets, n, seed,
                                                                                       out);
  return cudaGetLastError();
}

cudaError_t launch_hash_decimal(uint64_t start, uint64_t n, uint64_t seed, uint64_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  hash_decimal_kernel<<<static_cast<unsigned>(grid_for(n, 256, 148, 16)), 128, 0, s>>>(start, n, seed, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers (sbbf_internal.h)
// ---------------------------------------------------------------------------
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

template <typename K>
int resident_blocks(K kernel, int threads, size_t smem) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1)
    b = 1;
  return b;
}

uint64_t grid_for(uint64_t work_items, uint64_t items_per_block, int sms, int per_sm) {
  const uint64_t want = (work_items + items_per_block - 1) / items_per_block;
  const uint64_t cap = static_cast<uint64_t>(sms) * per_sm;
  uint64_t g = want < cap ? want : cap;
  return g < 1 ? 1 : g;
}

// Evict-last hints on the insert reds only pay where the filter competes for
// L2 (> L2 / 2); SBBF_RED_HINT=0/1 forces either (A/B only).
bool red_hint(const DeviceInfo& di, const Geom& g) {
  static const int force = [] {
    const char* v = getenv("SBBF_RED_HINT");
    return v ? atoi(v) : -1;
  }();
  if (force >= 0) return force != 0;
  return g.nb_local * 32 * 2 > static_cast<uint64_t>(di.l2_bytes);
}

// Range-split passes for a whole filter somewhat larger than L2: 2^k passes,
// each over every key but touching only one contiguous 1/2^k of the filter,
// which stays L2-resident while its keys land (config 3's 128 MiB filter:
// inserts 55.4 -> 113.6 Gkeys/s with 2 passes, 85.6 with 4; lookups 112.8
// (blocked) -> 137.6 with 2 passes, 69.2 with 4, whose extra hash-stream
// passes cost more than they save). Each range must fit in ~0.6 x L2.
bool split_compact() {  // SBBF_SPLIT_COMPACT=0 selects the uncompacted pass kernel (A/B only)
  static const bool on = [] {
    const char* v = getenv("SBBF_SPLIT_COMPACT");
    return !(v && v[0] == '0');
  }();
  return on;
}

int split_log2(const DeviceInfo& di, const Geom& g, bool lookup) {
  if (g.first != 0 || g.nb_local != g.nb_global) return 0;  // top hash bits = block ranges of a whole filter only
  const double part = 0.6 * static_cast<double>(di.l2_bytes);
  const double bytes = static_cast<double>(g.nb_local) * 32.0;
  if (bytes <= part) return 0;
  if (bytes <= 2 * part) return 1;
  return lookup || bytes > 4 * part ? 0 : 2;
}

cudaError_t launch_insert(const DeviceInfo& di, int variant, uint32_t* blocks, const Geom& g,
                          const uint64_t* hashes, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  if (variant == kInsertThread) {
    static const int occ = resident_blocks(insert_thread_kernel, kThreads, 0);
    const uint64_t grid = grid_for(n, kThreads * 4, di.sms, occ);
    insert_thread_kernel<<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
  } else if (variant == kInsertLane8Test) {
    static const int occ = resident_blocks(insert_lane8_kernel<true>, kThreads, 0);
    const uint64_t grid = grid_for(n, kThreads * 2, di.sms, occ);
    insert_lane8_kernel<true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
  } else if (variant == kInsertLane8) {
    static const int occ = resident_blocks(insert_lane8_kernel<false>, kThreads, 0);
    const uint64_t grid = grid_for(n, kThreads * 2, di.sms, occ);
    insert_lane8_kernel<false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
  } else if (variant == kInsertWideTest) {
    static const int occ = resident_blocks(insert_wide_kernel<true>, kThreads, 0);
    const uint64_t grid = grid_for(n, kThreads * 4, di.sms, occ);
    insert_wide_kernel<true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
  } else {
    // one warp step (4 x 32 keys) per warp, the grid covering the batch once:
    // the CTAs run in key order and each retires after one step (config 2
    // step 187.4 -> 188.6, config 3 inserts 51.9 -> 55.7 Gkeys/s vs a
    // persistent grid of 4 CTAs/SM)
    const uint64_t grid = (n + kThreads * 4 - 1) / (kThreads * 4);
    const int split_log = split_log2(di, g, false);
    if (split_log > 0) {
      for (uint64_t p = 0; p < (uint64_t{1} << split_log); ++p)
        insert_wide_kernel<false, false, 4, true, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(
            blocks, g, hashes, n, 0, static_cast<uint32_t>(64 - split_log), p);
    } else if (red_hint(di, g))
      insert_wide_kernel<false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
    else
      insert_wide_kernel<false, false, 4, false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g,
                                                                                                 hashes, n);
  }
  return cudaGetLastError();
}

cudaError_t launch_insert_ordered(const DeviceInfo& di, uint32_t* blocks, const Geom& g,
                                  const uint64_t* hashes, uint64_t n, bool test, cudaStream_t s) {
  (void)di;
  if (n == 0) return cudaSuccess;
  note_launch();
  const uint64_t grid = (n + kThreads * 4 - 1) / (kThreads * 4);  // 8 warps x 128 keys per CTA
  if (test)
    insert_wide_kernel<true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
  else
    insert_wide_kernel<false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, hashes, n);
  return cudaGetLastError();
}


// Fused XXH64 frontends: u64 keys hashed inside the insert / lookup kernel.
cudaError_t launch_insert_keys(const DeviceInfo& di, bool test, uint32_t* blocks, const Geom& g,
                               const uint64_t* keys, uint64_t n, uint64_t seed, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  if (test) {
    static const int occ = resident_blocks(insert_wide_kernel<true, true>, kThreads, 0);
    const uint64_t grid = grid_for(n, kThreads * 4, di.sms, occ);
    insert_wide_kernel<true, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, keys, n, seed);
  } else {
    const uint64_t grid = (n + kThreads * 4 - 1) / (kThreads * 4);  // as launch_insert's WIDE path
    const int split_log = split_log2(di, g, false);
    if (split_log > 0) {  // range-split passes, as launch_insert
      for (uint64_t p = 0; p < (uint64_t{1} << split_log); ++p)
        insert_wide_kernel<false, true, 4, true, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(
            blocks, g, keys, n, seed, static_cast<uint32_t>(64 - split_log), p);
    } else {
      insert_wide_kernel<false, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(blocks, g, keys, n, seed);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_find_keys(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const uint64_t* keys,
                             uint64_t n, uint64_t seed, void* out, bool bits, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  // the pipelined lookup with XXH64 applied to each key as it streams in,
  // launched like the raw-hash lookup (programmatic dependent of an insert)
  constexpr int kU = 4, kMinB = 3;
  static const int occ = resident_blocks(find_pipe_kernel<kU, true, kMinB, true>, kThreads, 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid_for(n, kThreads * kU, di.sms, occ)));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g.first == 0 && g.nb_local == g.nb_global) {  // a whole filter: the lean kernel, as for raw hashes
    static const int occ_w = resident_blocks(find_whole_kernel<kU, true, kMinB, true>, kThreads, 0);
    cfg.gridDim = dim3(static_cast<unsigned>(grid_for(n, kThreads * kU, di.sms, occ_w)));
    const int split_log = split_log2(di, g, true);
    if (split_log > 0) {  // range-split passes (XXH64 applied in each pass)
      cudaError_t e = cudaSuccess;
      for (uint64_t p = 0; p < (uint64_t{1} << split_log) && e == cudaSuccess; ++p) {
        const uint32_t psh = static_cast<uint32_t>(64 - split_log);
        e = bits ? cudaLaunchKernelEx(&cfg, find_whole_kernel<kU, true, kMinB, true, true>, blocks, g.nb_global, keys,
                                      n, out, seed, psh, p, p == 0)
                 : cudaLaunchKernelEx(&cfg, find_whole_kernel<kU, false, kMinB, true, true>, blocks, g.nb_global,
                                      keys, n, out, seed, psh, p, p == 0);
      }
      return e;
    }
    return bits ? cudaLaunchKernelEx(&cfg, find_whole_kernel<kU, true, kMinB, true>, blocks, g.nb_global, keys, n, out,
                                     seed, 63u, uint64_t{0}, true)
                : cudaLaunchKernelEx(&cfg, find_whole_kernel<kU, false, kMinB, true>, blocks, g.nb_global, keys, n,
                                     out, seed, 63u, uint64_t{0}, true);
  }
  return bits ? cudaLaunchKernelEx(&cfg, find_pipe_kernel<kU, true, kMinB, true>, blocks, g, keys, n, out, seed)
              : cudaLaunchKernelEx(&cfg, find_pipe_kernel<kU, false, kMinB, true>, blocks, g, keys, n, out, seed);
}
cudaError_t launch_find(const DeviceInfo& di, int variant, const uint32_t* blocks, const Geom& g,
                        const uint64_t* hashes, uint64_t n, void* out, bool bits, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  if (variant == kFindSmem) {
    const size_t smem = static_cast<size_t>(g.nb_local) * 32;
    auto kern = bits ? find_smem_kernel<true> : find_smem_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int threads = 1024;
    const uint64_t grid = grid_for(n, threads * 8, di.sms, 1);
    kern<<<static_cast<unsigned>(grid), threads, smem, s>>>(blocks, g, hashes, n, out);
  } else {
    // Pipelined lookup, 4 keys in flight per thread plus the next tile's
    // hashes, 3 CTAs/SM (sweep of U in {2,4,8} x CTAs/SM: profiles/r1_find_tuning.md).
    // Launched as a programmatic dependent of a preceding insert.
    constexpr int kU = 4, kMinB = 3;
    static const int occ = resident_blocks(find_pipe_kernel<kU, true, kMinB>, kThreads, 0);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (g.first == 0 && g.nb_local == g.nb_global) {  // a whole filter: the lean kernel
      static const int occ_w = resident_blocks(find_whole_kernel<kU, true, kMinB>, kThreads, 0);
      cfg.gridDim = dim3(static_cast<unsigned>(grid_for(n, kThreads * kU, di.sms, occ_w)));
      const int split_log = split_log2(di, g, true);
      if (split_log > 0) {
        constexpr int kUS = kU, kMinS = kMinB;  // U = 8 at 2 CTAs/SM measured the same (136.5 vs 137.6)
        static const int occ_s = resident_blocks(find_whole_kernel<kUS, true, kMinS, false, true>, kThreads, 0);
        cfg.gridDim = dim3(static_cast<unsigned>(grid_for(n, kThreads * kUS, di.sms, occ_s)));
        cudaError_t e = cudaSuccess;
        // Probes in flight per lane x CTAs per SM x keys per warp tile, config 3
        // (profiles/r2q_*): 2 x 4 x 256 (default) 159.6 Gkeys/s; 4 x 3 x 256
        // 147.9; 2 x 5 x 256 (spills) 106.6. SBBF_SPLIT_VARIANT selects others
        // (A/B only): 1 = 4x3x256, 3 = 1x6x128, 4 = 2x5x128, 5 = 2x6x128.
        static const int sv = [] {
          const char* v = getenv("SBBF_SPLIT_VARIANT");
          return v ? atoi(v) : 0;
        }();
        auto ksplit = sv == 0 ? find_split_kernel<2, 4> : sv == 3 ? find_split_kernel<1, 6, 128>
                      : sv == 4 ? find_split_kernel<2, 5, 128> : sv == 5 ? find_split_kernel<2, 6, 128>
                                                                 : find_split_kernel<4, 3>;
        const int tile = (sv == 3 || sv == 4 || sv == 5) ? 128 : 256;
        const int occ_c = resident_blocks(ksplit, kThreads, 0);
        // SBBF_SPLIT_PASSES (A/B only): compacted passes over equal ranges of
        // the top 32 hash bits (default 2^split_log)
        static const int np_env = [] {
          const char* v = getenv("SBBF_SPLIT_PASSES");
          const int x = v ? atoi(v) : 0;
          return x >= 2 && x <= 8 ? x : 0;
        }();
        const bool compact = bits && split_compact();
        const uint64_t passes = compact && np_env ? static_cast<uint64_t>(np_env) : uint64_t{1} << split_log;
        for (uint64_t p = 0; p < passes && e == cudaSuccess; ++p) {
          const bool first = p == 0;
          if (compact) {
            const uint64_t lo = (p << 32) / passes, hi = ((p + 1) << 32) / passes;
            cudaLaunchConfig_t cc = cfg;
            cc.gridDim = dim3(static_cast<unsigned>(grid_for(n, tile * (kThreads / 32), di.sms, occ_c)));
            e = cudaLaunchKernelEx(&cc, ksplit, blocks, g.nb_global, hashes, n, static_cast<uint32_t*>(out), lo,
                                   hi - lo, first);
          } else {
            const uint32_t psh = static_cast<uint32_t>(64 - split_log);
            e = bits ? cudaLaunchKernelEx(&cfg, find_whole_kernel<kUS, true, kMinS, false, true>, blocks, g.nb_global,
                                          hashes, n, out, uint64_t{0}, psh, p, first)
                     : cudaLaunchKernelEx(&cfg, find_whole_kernel<kUS, false, kMinS, false, true>, blocks,
                                          g.nb_global, hashes, n, out, uint64_t{0}, psh, p, first);
          }
        }
        return e;
      }
      return bits ? cudaLaunchKernelEx(&cfg, find_whole_kernel<kU, true, kMinB>, blocks, g.nb_global, hashes, n, out,
                                       uint64_t{0}, 63u, uint64_t{0}, true)
                  : cudaLaunchKernelEx(&cfg, find_whole_kernel<kU, false, kMinB>, blocks, g.nb_global, hashes, n, out,
                                       uint64_t{0}, 63u, uint64_t{0}, true);
    }
    cfg.gridDim = dim3(static_cast<unsigned>(grid_for(n, kThreads * kU, di.sms, occ)));  // a shard
    return bits ? cudaLaunchKernelEx(&cfg, find_pipe_kernel<kU, true, kMinB>, blocks, g, hashes, n, out, uint64_t{0})
                : cudaLaunchKernelEx(&cfg, find_pipe_kernel<kU, false, kMinB>, blocks, g, hashes, n, out, uint64_t{0});
  }
  return cudaGetLastError();
}

cudaError_t launch_block_index(const uint64_t* h, uint64_t n, uint64_t nb, uint64_t* out,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  const uint64_t grid = grid_for(n, 256, 148, 8);
  block_index_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(h, n, nb, out);
  return cudaGetLastError();
}

cudaError_t launch_make_mask(const uint64_t* h, uint64_t n, uint32_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  note_launch();
  const uint64_t grid = grid_for(n, 256, 148, 8);
  make_mask_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(h, n, out);
  return cudaGetLastError();
}

}  // namespace sbbf
