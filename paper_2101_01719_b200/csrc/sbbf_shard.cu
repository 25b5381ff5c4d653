// sbbf_shard.cu — key routing for the multi-GPU sharded filter.
//
// Rank r of P owns the contiguous global block range
// [floor(r*B/P), floor((r+1)*B/P)). Routing a batch is: count keys per owner
// (shard_count), exchange counts, scatter keys into per-owner segments
// (shard_scatter), all-to-all the segments (NCCL, in sharded.py), then the
// local insert/find kernels run with the shard's Geom. Lookup answers travel
// back in receive order and land in source order with scatter_u8.
//
// Both routing kernels work on CTA-sized chunks: a shared-memory histogram
// per chunk, one global atomic per (chunk, owner) to reserve output space,
// shared-memory atomics for slots inside the reservation. So global atomic
// traffic is P per 4096 keys, not one per key.
#include <cuda_runtime.h>

#include <cstdint>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

constexpr int kMaxParts = 1024;
constexpr int kShardThreads = 256;
constexpr int kPerThread = 16;
constexpr int kChunk = kShardThreads * kPerThread;

__device__ __forceinline__ uint32_t owner_of(uint64_t h, uint64_t total, const uint64_t* bounds,
                                             uint32_t parts) {
  const uint64_t b = dev::block_index(h, total);
  // last r with bounds[r] <= b
  uint32_t lo = 0, hi = parts - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (bounds[mid] <= b)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kShardThreads) shard_count_kernel(const uint64_t* __restrict__ hashes,
                                                                    uint64_t n, uint64_t total,
                                                                    const uint64_t* __restrict__ gbounds,
                                                                    uint32_t parts,
                                                                    unsigned long long* __restrict__ counts) {
  __shared__ uint64_t bounds[kMaxParts];
  __shared__ unsigned int hist[kMaxParts];
  for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) {
    bounds[i] = gbounds[i];
    hist[i] = 0;
  }
  __syncthreads();
  const uint64_t pol = dev::policy_evict_first();
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kChunk; base < n;
       base += static_cast<uint64_t>(gridDim.x) * kChunk) {
#pragma unroll 4
    for (int j = 0; j < kPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kShardThreads + threadIdx.x;
      if (i < n) atomicAdd(&hist[owner_of(dev::ld_stream_u64(hashes + i, pol), total, bounds, parts)], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x)
    if (hist[i]) atomicAdd(&counts[i], static_cast<unsigned long long>(hist[i]));
}

__global__ void __launch_bounds__(kShardThreads) shard_scatter_kernel(
    const uint64_t* __restrict__ hashes, uint64_t n, uint64_t total, const uint64_t* __restrict__ gbounds,
    uint32_t parts, unsigned long long* __restrict__ cursor, uint64_t* __restrict__ out,
    uint32_t* __restrict__ pos) {
  __shared__ uint64_t bounds[kMaxParts];
  __shared__ unsigned int hist[kMaxParts];
  __shared__ unsigned long long gbase[kMaxParts];
  for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) bounds[i] = gbounds[i];
  const uint64_t pol = dev::policy_evict_first();
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kChunk; base < n;
       base += static_cast<uint64_t>(gridDim.x) * kChunk) {
    for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    uint64_t h[kPerThread];
    uint32_t o[kPerThread];
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kShardThreads + threadIdx.x;
      if (i < n) {
        h[j] = dev::ld_stream_u64(hashes + i, pol);
        o[j] = owner_of(h[j], total, bounds, parts);
        atomicAdd(&hist[o[j]], 1u);
      } else {
        o[j] = 0xffffffffu;
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) {
      gbase[i] = hist[i] ? atomicAdd(&cursor[i], static_cast<unsigned long long>(hist[i])) : 0;
      hist[i] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      if (o[j] != 0xffffffffu) {
        const uint64_t slot = gbase[o[j]] + atomicAdd(&hist[o[j]], 1u);
        out[slot] = h[j];
        if (pos) pos[slot] = static_cast<uint32_t>(base + static_cast<uint64_t>(j) * kShardThreads + threadIdx.x);
      }
    }
    __syncthreads();
  }
}

__global__ void scatter_u8_kernel(const uint8_t* __restrict__ src, const uint32_t* __restrict__ pos,
                                  uint64_t n, uint8_t* __restrict__ dst) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    SBBF_DCHECK(pos[i] < n);
    dst[pos[i]] = src[i];
  }
}

__global__ void pack_bits_kernel(const uint8_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ bits) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t nw = (n + 31) / 32;
  // one warp-ballot per 32 keys
  for (uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += stride >> 5) {
    const uint64_t i = w * 32 + (threadIdx.x & 31);
    const uint32_t word = __ballot_sync(0xffffffffu, i < n && src[i] != 0);
    if ((threadIdx.x & 31) == 0) bits[w] = word;
  }
}

int shard_rc(cudaError_t e) { return e == cudaSuccess ? SBBF_OK : SBBF_ECUDA; }

// Exclusive prefix sum of parts (<= 1024) counts in one CTA.
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const unsigned long long* __restrict__ counts,
                                                              uint32_t parts,
                                                              unsigned long long* __restrict__ offsets) {
  __shared__ unsigned long long buf[2][kMaxParts];
  const uint32_t t = threadIdx.x;
  int cur = 0;
  buf[0][t] = (t > 0 && t <= parts) ? counts[t - 1] : 0ull;
  __syncthreads();
  for (uint32_t d = 1; d < kMaxParts; d <<= 1) {
    buf[cur ^ 1][t] = buf[cur][t] + (t >= d ? buf[cur][t - d] : 0ull);
    cur ^= 1;
    __syncthreads();
  }
  if (t < parts) offsets[t] = buf[cur][t];
}

}  // namespace

cudaError_t launch_partition(const uint64_t* hashes, uint64_t n, uint64_t total, const uint64_t* d_bounds,
                             uint32_t parts, uint64_t* d_counts, uint64_t* d_offsets, uint64_t* d_cursor,
                             uint64_t* d_out, uint32_t* d_pos, int sms, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_counts, 0, parts * sizeof(uint64_t), s);
  if (e != cudaSuccess || n == 0) return e;
  const uint64_t grid = grid_for(n, kChunk, sms, 8);
  note_launch();
  shard_count_kernel<<<static_cast<unsigned>(grid), kShardThreads, 0, s>>>(
      hashes, n, total, d_bounds, parts, reinterpret_cast<unsigned long long*>(d_counts));
  note_launch();
  exclusive_scan_kernel<<<1, kMaxParts, 0, s>>>(reinterpret_cast<unsigned long long*>(d_counts), parts,
                                                reinterpret_cast<unsigned long long*>(d_offsets));
  e = cudaMemcpyAsync(d_cursor, d_offsets, parts * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  note_launch();
  shard_scatter_kernel<<<static_cast<unsigned>(grid), kShardThreads, 0, s>>>(
      hashes, n, total, d_bounds, parts, reinterpret_cast<unsigned long long*>(d_cursor), d_out, d_pos);
  return cudaGetLastError();
}

}  // namespace sbbf

extern "C" {

int sbbf_shard_bounds(uint64_t total_buckets, uint32_t parts, uint64_t* h_bounds) {
  if (!h_bounds || parts == 0 || parts > sbbf::kMaxParts || total_buckets < parts) return SBBF_EINVAL;
  for (uint32_t r = 0; r <= parts; ++r)
    h_bounds[r] = static_cast<uint64_t>((static_cast<unsigned __int128>(total_buckets) * r) / parts);
  return SBBF_OK;
}

int sbbf_shard_count(const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                     const uint64_t* d_bounds, uint32_t parts, uint64_t* d_counts, void* stream) {
  if (!d_counts || !d_bounds || parts == 0 || parts > sbbf::kMaxParts || (n && !d_hashes))
    return SBBF_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_counts, 0, parts * sizeof(uint64_t), s);
  if (e != cudaSuccess || n == 0) return sbbf::shard_rc(e);
  sbbf::note_launch();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t grid = sbbf::grid_for(n, sbbf::kChunk, sms, 8);
  sbbf::shard_count_kernel<<<static_cast<unsigned>(grid), sbbf::kShardThreads, 0, s>>>(
      d_hashes, n, total_buckets, d_bounds, parts, reinterpret_cast<unsigned long long*>(d_counts));
  return sbbf::shard_rc(cudaGetLastError());
}

int sbbf_shard_scatter(const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                       const uint64_t* d_bounds, uint32_t parts, const uint64_t* d_offsets,
                       uint64_t* d_cursor, uint64_t* d_out, uint32_t* d_pos, void* stream) {
  if (!d_bounds || !d_offsets || !d_cursor || parts == 0 || parts > sbbf::kMaxParts ||
      (n && (!d_hashes || !d_out)) || n > 0xffffffffull)
    return SBBF_EINVAL;
  if (n == 0) return SBBF_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(d_cursor, d_offsets, parts * sizeof(uint64_t),
                                  cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return sbbf::shard_rc(e);
  sbbf::note_launch();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t grid = sbbf::grid_for(n, sbbf::kChunk, sms, 8);
  sbbf::shard_scatter_kernel<<<static_cast<unsigned>(grid), sbbf::kShardThreads, 0, s>>>(
      d_hashes, n, total_buckets, d_bounds, parts, reinterpret_cast<unsigned long long*>(d_cursor), d_out,
      d_pos);
  return sbbf::shard_rc(cudaGetLastError());
}

int sbbf_shard_partition(const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                         const uint64_t* d_bounds, uint32_t parts, uint64_t* d_counts, uint64_t* d_scratch,
                         uint64_t* d_out, uint32_t* d_pos, void* stream) {
  if (!d_bounds || !d_counts || !d_scratch || parts == 0 || parts > 64 || (n && (!d_hashes || !d_out)) ||
      n > 0xffffffffull)
    return SBBF_EINVAL;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sbbf::DeviceInfo di;
  di.device = dev;
  di.sms = sms;
  return sbbf::shard_rc(sbbf::shard_partition(di, total_buckets, parts, d_bounds, d_hashes, n, d_counts,
                                              d_scratch, d_out, d_pos, static_cast<cudaStream_t>(stream)));
}

int sbbf_scatter_u8(const uint8_t* d_src, const uint32_t* d_pos, uint64_t n, uint8_t* d_dst,
                    void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_src || !d_pos || !d_dst) return SBBF_EINVAL;
  sbbf::note_launch();
  const uint64_t grid = sbbf::grid_for(n, 1024, 148, 16);
  sbbf::scatter_u8_kernel<<<static_cast<unsigned>(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_src, d_pos, n, d_dst);
  return sbbf::shard_rc(cudaGetLastError());
}

int sbbf_pack_bits(const uint8_t* d_src, uint64_t n, uint32_t* d_bits, void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_src || !d_bits) return SBBF_EINVAL;
  sbbf::note_launch();
  const uint64_t grid = sbbf::grid_for(n, 256, 148, 16);
  sbbf::pack_bits_kernel<<<static_cast<unsigned>(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_src, n, d_bits);
  return sbbf::shard_rc(cudaGetLastError());
}

}  // extern "C"
