// microbench_dsmem.cu — distributed shared memory throughput inside an
// 8-CTA cluster on B200 (design evidence for a cluster-partitioned lookup).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o scripts/bin/microbench_dsmem scripts/microbench_dsmem.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int kSlots = 16384;  // 128 KiB of u64 per CTA

__device__ __forceinline__ uint32_t xs(uint32_t x) {
  x ^= x << 13;
  x ^= x >> 17;
  return x ^ (x << 5);
}

// MODE 0: remote 8-byte stores to random CTA/slot; 1: same but local CTA only;
// 2: remote 32-byte loads (2 x v4); 3: local 32-byte loads
template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 1) dsmem_kernel(int iters, uint64_t* sink) {
  extern __shared__ __align__(16) uint64_t buf[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) buf[i] = i;
  cl.sync();
  uint32_t r = 0x9E3779B9u ^ (blockIdx.x * 1024 + threadIdx.x);
  uint64_t acc = 0;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  for (int it = 0; it < iters; ++it) {
    r = xs(r);
    const uint32_t dst = (MODE == 1 || MODE == 3) ? cl.block_rank() : (r & 7u);
    const uint32_t slot = (r >> 3) & (kSlots - 4);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + slot * 8), "r"(dst));
    if constexpr (MODE <= 1) {
      asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(static_cast<uint64_t>(r)) : "memory");
    } else {
      uint32_t a, b, c, d, e, f, g, h;
      asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                   : "r"(ra));
      asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4+16];"
                   : "=r"(e), "=r"(f), "=r"(g), "=r"(h)
                   : "r"(ra));
      acc += a ^ b ^ c ^ d ^ e ^ f ^ g ^ h;
    }
  }
  cl.sync();
  if (acc == 0x12345) sink[0] = acc;
}

template <int MODE>
void run(const char* name, int sms) {
  const int clusters = sms / 8;
  const int iters = 1 << 14;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * 8 * 2);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = kSlots * 8;
  CK(cudaFuncSetAttribute(dsmem_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * 8));
  uint64_t* sink;
  CK(cudaMalloc(&sink, 64));
  int nclusters = 0;
  cudaLaunchConfig_t q = cfg;
  CK(cudaOccupancyMaxActiveClusters(&nclusters, dsmem_kernel<MODE>, &q));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaLaunchKernelEx(&cfg, dsmem_kernel<MODE>, iters, sink));
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  CK(cudaLaunchKernelEx(&cfg, dsmem_kernel<MODE>, iters, sink));
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double ops = double(cfg.gridDim.x) * 512 * iters;
  printf("%-26s max active clusters %3d  %8.2f G ops/s  (%.3f ops/clk/SM at 1.965 GHz over %d SMs)\n", name,
         nclusters, ops / ms / 1e6, ops / (ms * 1e-3) / 1.965e9 / (nclusters * 8), nclusters * 8);
  CK(cudaFree(sink));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<0>("remote st.u64", sms);
  run<1>("local  st.u64 (cluster)", sms);
  run<2>("remote ld 32B", sms);
  run<3>("local  ld 32B (cluster)", sms);
  return 0;
}
