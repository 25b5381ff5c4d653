// Shared-memory atomic OR throughput on sm_100a: random 64-bit / 32-bit
// atom.shared.or over a 128 KiB table (the smem-tile insert's apply step),
// with and without test-before-set. Lane-ops per SM-clock.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/bin/microbench_smem_atom scripts/microbench_smem_atom.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kWords = 128 * 1024 / 8;  // 16K u64
constexpr int kIters = 4096;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; return x ^ (x >> 33);
}

template <int M>  // 0: atom.or.b64, 1: atom.or.b32 x2, 2: test + atom.or.b64, 3: plain ld/st (racy, reference)
__global__ void __launch_bounds__(1024, 1) kern(uint64_t* out, uint64_t seed) {
  extern __shared__ uint64_t t[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) t[i] = 0;
  __syncthreads();
  uint64_t x = mix(seed + blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < kIters; ++it) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    const uint32_t w = static_cast<uint32_t>(x >> 40) & (kWords - 1);
    const uint64_t m = (1ull << ((x >> 8) & 63)) | (1ull << ((x >> 16) & 63));
    if (M == 0) atomicOr(reinterpret_cast<unsigned long long*>(&t[w]), m);
    if (M == 1) {
      atomicOr(reinterpret_cast<unsigned*>(&t[w]), static_cast<unsigned>(m));
      atomicOr(reinterpret_cast<unsigned*>(&t[w]) + 1, static_cast<unsigned>(m >> 32));
    }
    if (M == 2) {
      if (m & ~t[w]) atomicOr(reinterpret_cast<unsigned long long*>(&t[w]), m);
    }
    if (M == 3) t[w] |= m;
  }
  __syncthreads();
  uint64_t acc = 0;
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) acc ^= t[i];
  if (acc == 0x1234) out[0] = acc;
}

template <int M>
void run(const char* name, int sms) {
  uint64_t* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(kern<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<M><<<sms, 1024, kWords * 8>>>(out, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<M><<<sms, 1024, kWords * 8>>>(out, r + 2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = 5.0 * sms * 1024.0 * kIters;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-28s %8.2f G lane-ops/s  %6.2f lane-ops/clk/SM (at %d MHz)  %s\n", name, ops / ms / 1e6,
         ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("atom.shared.or.b64", sms);
  run<1>("atom.shared.or.b32 x2", sms);
  run<2>("test + atom.shared.or.b64", sms);
  run<3>("ld/st shared (racy ref)", sms);
  return 0;
}
