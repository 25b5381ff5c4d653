// sbbf_probe.cu — random 32-byte-sector microbenchmarks: the roofline
// denominators for the metric "Gkeys/s vs random-32B-sector roofline".
//
// Both kernels draw block indices from splitmix64 in registers (no hash
// stream), so they measure only the random-sector path the SBBF kernels
// share: one 256-bit LDG per key (sector_read) or one 32-byte atomic-OR
// sector op per key via the inserts' own pattern, 4 lanes x red.b64 (L1
// merges them into one sector request; sector_red). Run on a buffer larger
// than L2 they give the HBM random-sector ceiling; on a 1 MiB buffer, the L2
// one.
#include <cuda_runtime.h>

#include <cstdint>

#include "sbbf_bench.h"
#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <int U>
__global__ void __launch_bounds__(256, 4) sector_read_kernel(const uint32_t* __restrict__ buf,
                                                             uint64_t nb, uint64_t n, uint64_t seed,
                                                             uint32_t* __restrict__ sink) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t base = tid; base < n; base += stride * U) {
    dev::Block8 b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = base + u * stride;
      const uint64_t h = mix(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
      dev::ld_block_nc(buf + dev::block_index(h, nb) * 8, b[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * stride < n) {
#pragma unroll
        for (int w = 0; w < 8; ++w) acc ^= b[u].w[w];
      }
    }
  }
  if (acc == 0x9e3779b9u) sink[tid & 1023] = acc;  // keeps the loads live
}

__global__ void __launch_bounds__(256, 4) sector_red_kernel(uint32_t* __restrict__ buf, uint64_t nb,
                                                            uint64_t n, uint64_t seed) {
  // insert_wide_kernel's pattern: 4 threads per key, one red.b64 per lane
  // pair (no cache hint, as its L2-resident launch)
  const int lane = threadIdx.x & 31;
  const int pair = lane & 3;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t t = warp; t * 32 < n; t += nwarps) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t k = t * 32 + r * 8 + (lane >> 2);
      if (k < n) {
        const uint64_t h = mix(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
        const uint64_t m = (uint64_t{1} << (h & 31)) | (uint64_t{1} << (32 + ((h >> 5) & 31)));
        dev::red_or64_nohint(reinterpret_cast<uint64_t*>(buf + dev::block_index(h, nb) * 8) + pair, m);
      }
    }
  }
}

}  // namespace
}  // namespace sbbf

extern "C" {

int sbbf_bench_sector_read(const uint32_t* d_buf, uint64_t num_blocks, uint64_t n, uint64_t seed,
                           uint32_t* d_sink, void* stream) {
  if (!d_buf || !d_sink || num_blocks == 0) return SBBF_EINVAL;
  if (n == 0) return SBBF_OK;
  sbbf::note_launch();
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sbbf::sector_read_kernel<8><<<sms * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_buf, num_blocks, n, seed, d_sink);
  return cudaGetLastError() == cudaSuccess ? SBBF_OK : SBBF_ECUDA;
}

int sbbf_bench_sector_red(uint32_t* d_buf, uint64_t num_blocks, uint64_t n, uint64_t seed,
                          void* stream) {
  if (!d_buf || num_blocks == 0) return SBBF_EINVAL;
  if (n == 0) return SBBF_OK;
  sbbf::note_launch();
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sbbf::sector_red_kernel<<<sms * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_buf, num_blocks,
                                                                                   n, seed);
  return cudaGetLastError() == cudaSuccess ? SBBF_OK : SBBF_ECUDA;
}

}  // extern "C"
