// sbbf_mc.cu — Monte-Carlo false-positive oracle at scale: the reference's
// sbbf_fpp_mc (core/src/model.cpp:105-128) on the GPU.
//
// The reference fills every block with Poisson(a) hashes drawn uniformly from
// that block's preimage interval [b*2^64/B, (b+1)*2^64/B) (Knuth inversion,
// hash_for_bucket: floor((b*2^64 + r)/B), model.cpp:20-58) and probes
// `trials` uniform hashes. Its sampler is one sequential mt19937_64 stream,
// which does not parallelise, so this oracle keeps the same distributions
// with a counter-based stream per block (splitmix64 seeded by (seed, b)):
// statistically the same experiment, seed-reproducible, not the same draws.
// Validated like the reference validates its own (model_test.cpp:174-207):
// empty filters never hit, reproducible per seed, within 3 binomial standard
// errors of the series sbbf_fpp(a), identical input errors.
//
// Each thread owns whole blocks: the Poisson keys of block b are ORed into
// registers and the block is stored once (no atomics), so a 2^28-block (8 GiB)
// filter at a ~ 24 (6.4e9 keys) fills in one pass over HBM.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Stream {  // splitmix64 seeded per (seed, block)
  uint64_t s;
  __device__ explicit Stream(uint64_t seed, uint64_t b) : s(fmix64(seed ^ fmix64(b + 0x632be59bd9b4e019ull))) {}
  __device__ __forceinline__ uint64_t next() { return fmix64(s += 0x9e3779b97f4a7c15ull); }
  __device__ __forceinline__ double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

__global__ void mc_fill_kernel(uint32_t* __restrict__ blocks, uint64_t nb, double a, double limit, uint64_t seed) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < nb; b += stride) {
    Stream rng(seed, b);
    uint32_t lanes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (a > 0.0) {
      // poisson_sample (model.cpp:24-33): Knuth inversion
      uint64_t count = 0;
      double product = rng.uniform01();
      while (product > limit) {
        ++count;
        product *= rng.uniform01();
      }
      for (uint64_t i = 0; i < count; ++i) {
        // hash_for_bucket (model.cpp:38-48)
        const unsigned __int128 numer = (static_cast<unsigned __int128>(b) << 64) | rng.next();
        uint64_t h = static_cast<uint64_t>(numer / nb);
        while (dev::block_index(h, nb) != b) ++h;
        const uint32_t low = static_cast<uint32_t>(h);
#pragma unroll
        for (int w = 0; w < 8; ++w) lanes[w] |= dev::lane_bit(low, dev::lane_seed(w));
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(blocks + b * 8);
    dst[0] = make_uint4(lanes[0], lanes[1], lanes[2], lanes[3]);
    dst[1] = make_uint4(lanes[4], lanes[5], lanes[6], lanes[7]);
  }
}

__global__ void mc_probe_kernel(const uint32_t* __restrict__ blocks, uint64_t nb, uint64_t trials, uint64_t seed,
                                unsigned long long* __restrict__ hits) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const Stream base(seed, ~uint64_t{0});  // the probe stream: its own counter space
  uint64_t mine = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < trials; i += stride) {
    const uint64_t h = fmix64(base.s + (i + 1) * 0x9e3779b97f4a7c15ull);
    dev::Block8 blk;
    dev::ld_block_nc(blocks + dev::block_index(h, nb) * 8, blk);
    mine += dev::block_contains(blk, h) ? 1 : 0;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, d);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(hits, static_cast<unsigned long long>(mine));
}

}  // namespace
}  // namespace sbbf

extern "C" {

int sbbf_gpu_fpp_mc(double a, uint64_t blocks, uint64_t trials, uint64_t seed, int device, double* fpp) {
  // check_a + the oracle's own bounds (model.cpp:61-68, 106-112)
  if (!fpp || !std::isfinite(a) || a < 0.0 || a > 1e6) {
    sbbf::set_last_error("per-block density a must be finite, nonnegative and <= 1e6");
    return SBBF_EINVAL;
  }
  if (blocks < 1 || trials < 1) {
    sbbf::set_last_error("sbbf_fpp_mc needs at least one block and one trial");
    return SBBF_EINVAL;
  }
  if (a > 500.0) {
    sbbf::set_last_error("sbbf_fpp_mc supports densities up to 500");
    return SBBF_EINVAL;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    sbbf::set_last_error("sbbf_gpu_fpp_mc: no CUDA device (there is no CPU fallback)");
    return SBBF_ENODEV;
  }
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint32_t* d_blocks = nullptr;
  unsigned long long* d_hits = nullptr;
  cudaError_t e = cudaMalloc(&d_blocks, blocks * 32);
  if (e == cudaSuccess) e = cudaMalloc(&d_hits, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(d_hits, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) {
    sbbf::note_launch();
    sbbf::mc_fill_kernel<<<static_cast<unsigned>(sbbf::grid_for(blocks, 256, sms, 8)), 256>>>(
        d_blocks, blocks, a, std::exp(-a), seed);
    sbbf::note_launch();
    sbbf::mc_probe_kernel<<<static_cast<unsigned>(sbbf::grid_for(trials, 256 * 8, sms, 8)), 256>>>(
        d_blocks, blocks, trials, seed, d_hits);
    e = cudaGetLastError();
  }
  unsigned long long hits = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&hits, d_hits, sizeof(hits), cudaMemcpyDeviceToHost);
  cudaFree(d_blocks);
  cudaFree(d_hits);
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    sbbf::set_last_error(std::string("sbbf_gpu_fpp_mc: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SBBF_ENOMEM : SBBF_ECUDA;
  }
  *fpp = static_cast<double>(hits) / static_cast<double>(trials);
  return SBBF_OK;
}

}  // extern "C"
