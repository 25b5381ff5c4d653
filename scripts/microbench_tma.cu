// microbench_tma.cu — random 32-byte block fetches through the async copy
// engines instead of the LSU (design evidence; not part of the product).
//
//   A  cp.async.bulk (1-D, 32 B per key, one instruction per key)
//   B  cp.async.bulk.tensor.2d tile, box {8 u32, 1 row}, one per key
//   C  cp.async.bulk.tensor.2d tile::gather4, 4 random rows per instruction
// B and C run with the tensor map's L2 promotion NONE and 128B, to see
// whether DRAM fills shrink to the 32-byte sector.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o scripts/bin/microbench_tma scripts/microbench_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

constexpr int kStages = 4;
constexpr int kWarps = 8;

// MODE 0: bulk 1D; 1: tensor tile per key; 2: gather4
template <int MODE>
__global__ void __launch_bounds__(256, 1) tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                     const uint32_t* __restrict__ buf, uint64_t nb,
                                                     uint64_t n, uint64_t seed, uint32_t* sink) {
  __shared__ __align__(128) uint32_t stage[kWarps][kStages][32 * 8];
  __shared__ __align__(8) uint64_t bars[kWarps][kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) mbar_init(smem_u32(&bars[warp][s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarps;
  const uint64_t nbatch = n / 32;
  uint32_t acc = 0;
  uint32_t phase[kStages] = {0, 0, 0, 0};

  auto issue = [&](uint64_t b, int s) {
    const uint64_t k = b * 32 + lane;
    const uint64_t h = mix(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
    const uint32_t row = static_cast<uint32_t>(__umul64hi(h, nb));
    const uint32_t bar = smem_u32(&bars[warp][s]);
    if (lane == 0) mbar_expect(bar, 32 * 32);
    __syncwarp();
    const uint32_t dst = smem_u32(&stage[warp][s][lane * 8]);
    if constexpr (MODE == 0) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];" ::"r"(dst),
          "l"(buf + static_cast<uint64_t>(row) * 8), "r"(bar)
          : "memory");
    } else if constexpr (MODE == 1) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              dst),
          "l"(&tmap), "r"(0), "r"(row), "r"(bar)
          : "memory");
    } else {
      const uint32_t r0 = __shfl_sync(0xffffffffu, row, (lane & ~3) + 0);
      const uint32_t r1 = __shfl_sync(0xffffffffu, row, (lane & ~3) + 1);
      const uint32_t r2 = __shfl_sync(0xffffffffu, row, (lane & ~3) + 2);
      const uint32_t r3 = __shfl_sync(0xffffffffu, row, (lane & ~3) + 3);
      if ((lane & 3) == 0)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                dst),
            "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
            : "memory");
    }
  };

  uint64_t b = gwarp;
  for (int s = 0; s < kStages; ++s)
    if (b + s * nwarps < nbatch) issue(b + s * nwarps, s);
  for (uint64_t i = 0; b < nbatch; ++i, b += nwarps) {
    const int s = static_cast<int>(i % kStages);
    mbar_wait(smem_u32(&bars[warp][s]), phase[s]);
    phase[s] ^= 1;
    const uint4 lo = *reinterpret_cast<const uint4*>(&stage[warp][s][lane * 8]);
    const uint4 hi = *reinterpret_cast<const uint4*>(&stage[warp][s][lane * 8 + 4]);
    acc ^= lo.x ^ lo.y ^ lo.z ^ lo.w ^ hi.x ^ hi.y ^ hi.z ^ hi.w;
    __syncwarp();
    const uint64_t nb2 = b + kStages * nwarps;
    if (nb2 < nbatch) issue(nb2, s);
  }
  if (acc == 0x9e3779b9u) sink[threadIdx.x] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeTiled encode = reinterpret_cast<EncodeTiled>(fn);
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4096));
  const uint64_t n = 1ull << 26;
  const uint64_t sizes[] = {1, 1024, 4096};
  for (uint64_t mib : sizes) {
    uint32_t* buf;
    const uint64_t nb = (mib << 20) / 32;
    CK(cudaMalloc(&buf, mib << 20));
    CK(cudaMemset(buf, 0, mib << 20));
    for (int promo = 0; promo < 2; ++promo) {
      for (int boxrows = 1; boxrows <= 1; boxrows += 3) {
        CUtensorMap tm;
        cuuint64_t gdim[2] = {8, nb};
        cuuint64_t gstride[1] = {32};
        cuuint32_t box[2] = {8, static_cast<cuuint32_t>(boxrows)};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, gdim, gstride, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("encode failed promo=%d boxrows=%d: %d\n", promo, boxrows, (int)r);
          continue;
        }
        auto run = [&](auto kern, const char* name) {
          cudaEvent_t a, b;
          CK(cudaEventCreate(&a));
          CK(cudaEventCreate(&b));
          kern<<<sms * 2, 256>>>(tm, buf, nb, n, 1, sink);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("%-10s buf=%5llu MiB promo=%d box=%d: ERROR %s\n", name, (unsigned long long)mib, promo,
                   boxrows, cudaGetErrorString(e));
            exit(2);
          }
          float best = 1e30f;
          for (int i = 0; i < 3; ++i) {
            CK(cudaEventRecord(a));
            kern<<<sms * 2, 256>>>(tm, buf, nb, n, 7 + i, sink);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = ms < best ? ms : best;
          }
          printf("%-10s buf=%5llu MiB promo=%s box=%d  %8.2f G keys/s\n", name, (unsigned long long)mib,
                 promo ? "128B" : "none", boxrows, n / best / 1e6);
          fflush(stdout);
        };
        // (tile mode needs 128-byte aligned smem rows; a per-key tile load is
        // not run here — bulk1d already shows the per-request cost)
        if (boxrows == 1 && promo == 0) run(tma_kernel<0>, "bulk1d");
        run(tma_kernel<2>, "gather4");
      }
    }
    CK(cudaFree(buf));
  }
  return 0;
}
