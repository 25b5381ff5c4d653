// sbbf_blocked.cu — L2-blocked insert/lookup for filters larger than L2.
//
// A random 32-byte probe that misses L2 costs a full DRAM line fill
// (ncu: ~117 B of DRAM per key on a 1 GiB filter) and the HBM random-sector
// rate tops out at 37-43 G/s whatever the access path (LSU, TMA, gather4;
// profiles/r1_microbench_*.log). The blocked path trades that for streaming:
//
//   1. partition the batch by filter slice (launch_partition: CTA-chunked
//      histogram + reservation scatter, 8 B in / 12 B out per key),
//   2. process the grouped keys in slice order — CTAs are dispatched in
//      blockIdx order, so the keys in flight at any moment fall in one or two
//      slices (<= ~24 MiB each) and their probes/atomics hit L2; every filter
//      line is fetched from HBM about once per chunk,
//   3. lookups set their answer bit at the key's source position with a red
//      into a chunk bitmap that stays L2-resident.
//
// Per-key HBM traffic ~ 8 (read) + 12 (grouped write) + 12 (grouped read)
// + filter_bytes / chunk_keys, instead of a ~128-byte random line fill.
#include <cuda_runtime.h>

#include <cstdint>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

constexpr uint64_t kBlockedChunk = uint64_t{1} << 28;  // keys per partition round (3.1 GB scratch)
constexpr int kProbeU = 8;
constexpr int kProbeThreads = 256;
constexpr uint64_t kProbeTile = kProbeThreads * kProbeU;

__global__ void __launch_bounds__(kProbeThreads, 2) probe_grouped_kernel(
    const uint32_t* __restrict__ blocks, Geom g, const uint64_t* __restrict__ keys,
    const uint32_t* __restrict__ pos, uint64_t m, uint32_t* __restrict__ bitmap) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kProbeTile + threadIdx.x;
  const uint64_t pol = dev::policy_evict_first();
  uint64_t h[kProbeU];
  uint32_t p[kProbeU];
#pragma unroll
  for (int u = 0; u < kProbeU; ++u) {
    const uint64_t i = base + static_cast<uint64_t>(u) * kProbeThreads;
    h[u] = i < m ? dev::ld_stream_u64(keys + i, pol) : 0;
    p[u] = i < m ? pos[i] : 0;
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
      atomicOr(bitmap + (p[u] >> 5), 1u << (p[u] & 31));
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
  uint64_t* counts = nullptr;  // [3][parts]: counts, offsets, cursor
  uint32_t* bits = nullptr;
};

cudaError_t alloc_scratch(Scratch& sc, uint64_t cap, uint32_t parts, bool with_pos, bool with_bits,
                          cudaStream_t s) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sc.keys), cap * sizeof(uint64_t), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&sc.counts), 3 * parts * sizeof(uint64_t), s);
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

cudaError_t blocked_insert(const DeviceInfo& di, uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                           const uint64_t* hashes, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t cap = n < kBlockedChunk ? n : kBlockedChunk;
  Scratch sc;
  cudaError_t e = alloc_scratch(sc, cap, plan.parts, false, false, s);
  for (uint64_t off = 0; e == cudaSuccess && off < n; off += cap) {
    const uint64_t m = n - off < cap ? n - off : cap;
    e = launch_partition(hashes + off, m, g.nb_global, plan.d_bounds, plan.parts, sc.counts,
                         sc.counts + plan.parts, sc.counts + 2 * plan.parts, sc.keys, nullptr, di.sms, s);
    if (e == cudaSuccess) e = launch_insert_ordered(di, blocks, g, sc.keys, m, s);
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
      e = launch_partition(hashes + off, m, g.nb_global, plan.d_bounds, plan.parts, sc.counts,
                           sc.counts + plan.parts, sc.counts + 2 * plan.parts, sc.keys, sc.pos, di.sms, s);
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
