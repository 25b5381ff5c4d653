// microbench_zerocopy.cu — can the host-buffer path read hashes straight
// from pinned host memory (zero-copy over PCIe) faster than the DMA-staged
// pipeline? Design evidence only; not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/microbench_zerocopy scripts/microbench_zerocopy.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// U independent 16-byte loads per thread per step (grid-stride).
template <int U>
__global__ void read_kernel(const uint4* __restrict__ p, uint64_t n16, uint64_t* sink) {
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t i = tid; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n16 ? p[i + u * stride] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <typename L>
float best_ms(L f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r >= 2) best = std::min(best, ms);
  }
  return best;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t bytes = 88000000;  // config 2's hashes per step
  void* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  memset(h, 1, bytes);
  void* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  void* d;
  CK(cudaMalloc(&d, bytes));
  uint64_t* sink;
  CK(cudaMalloc(&sink, 8));
  float ms = best_ms([&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice)); });
  printf("cudaMemcpyAsync H2D 88 MB             %7.3f ms  %6.1f GB/s\n", ms, bytes / ms / 1e6);
  const uint64_t n16 = bytes / 16;
  for (int per_sm : {2, 4, 8, 16}) {
    ms = best_ms([&] { read_kernel<4><<<sms * per_sm, 256>>>(static_cast<const uint4*>(hd), n16, sink); });
    printf("zero-copy kernel read, %2d CTAs/SM U=4 %7.3f ms  %6.1f GB/s\n", per_sm, ms, bytes / ms / 1e6);
    ms = best_ms([&] { read_kernel<8><<<sms * per_sm, 256>>>(static_cast<const uint4*>(hd), n16, sink); });
    printf("zero-copy kernel read, %2d CTAs/SM U=8 %7.3f ms  %6.1f GB/s\n", per_sm, ms, bytes / ms / 1e6);
  }
  return 0;
}
