// microbench.cu — random 32-byte sector access flavours on B200 (design
// evidence for the SBBF kernels; not part of the product).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/microbench scripts/microbench.cu
//   scripts/bin/microbench            # prints one line per (flavour, buffer size)
//
// Every kernel draws block indices from splitmix64 in registers, so only the
// random-sector path is measured. Rates are G keys (sectors) per second.
#include <cuda.h>
#include <cuda_runtime.h>

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

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t key_hash(uint64_t seed, uint64_t k) {
  return mix(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
}

struct V8 {
  uint32_t w[8];
};

template <int F>
__device__ __forceinline__ void load32(const uint32_t* p, V8& b) {
  if constexpr (F == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 1) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 2) {
    asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 3) {
    asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 4) {
    asm volatile("ld.global.cs.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 5) {
    asm volatile("ld.global.cv.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 6) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%8];\n\t"
        "ld.global.nc.L1::no_allocate.v4.u32 {%4,%5,%6,%7}, [%8+16];"
        : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
          "=r"(b.w[6]), "=r"(b.w[7])
        : "l"(p));
  } else if constexpr (F == 7) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else if constexpr (F == 8) {
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(b.w[0]) : "l"(p));
#pragma unroll
    for (int i = 1; i < 8; ++i) b.w[i] = 0;
  } else if constexpr (F == 9) {
    asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  }
}

template <int F>
__global__ void __launch_bounds__(256, 4) read_kernel(const uint32_t* __restrict__ buf, uint64_t nb,
                                                      uint64_t n, uint64_t seed, uint32_t* sink) {
  constexpr int U = 8;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t base = tid; base < n; base += stride * U) {
    V8 b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) load32<F>(buf + __umul64hi(key_hash(seed, base + u * stride), nb) * 8, b[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int w = 0; w < 8; ++w) acc ^= b[u].w[w];
  }
  if (acc == 0x9e3779b9u) sink[tid & 1023] = acc;
}

// R: 0 = 8 x red.b32 lane-parallel (8 thr/key); 1 = 4 x red.b64 (4 thr/key);
//    2 = 8 x red.b32 one thread per key; 3 = atom.or.b32 lane-parallel (returning)
//    4 = 2 x red.b64 ... no: 4 = ld.lane then red only if missing (test-before-set, lane8)
template <int R>
__global__ void __launch_bounds__(256, 4) red_kernel(uint32_t* __restrict__ buf, uint64_t nb, uint64_t n,
                                                     uint64_t seed) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  if constexpr (R == 0 || R == 3 || R == 4) {
    const int word = lane & 7;
    for (uint64_t t = warp; t * 32 < n; t += nwarps) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint64_t k = t * 32 + r * 4 + (lane >> 3);
        const uint64_t h = key_hash(seed, k);
        uint32_t* p = buf + __umul64hi(h, nb) * 8 + word;
        const uint32_t bit = 1u << ((h >> (5 * word)) & 31);
        if constexpr (R == 0) {
          asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(bit) : "memory");
        } else if constexpr (R == 3) {
          uint32_t old;
          asm volatile("atom.relaxed.gpu.global.or.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(bit) : "memory");
          if (old == 0x12345u) buf[0] = old;
        } else {
          uint32_t cur;
          asm volatile("ld.global.u32 %0, [%1];" : "=r"(cur) : "l"(p));
          if (!(cur & bit)) asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(bit) : "memory");
        }
      }
    }
  } else if constexpr (R == 1) {
    const int word = lane & 3;
    for (uint64_t t = warp; t * 32 < n; t += nwarps) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint64_t k = t * 32 + r * 8 + (lane >> 2);
        const uint64_t h = key_hash(seed, k);
        uint64_t* p = reinterpret_cast<uint64_t*>(buf + __umul64hi(h, nb) * 8) + word;
        const uint64_t m = (1ull << ((h >> (10 * word)) & 31)) | (1ull << (32 + ((h >> (10 * word + 5)) & 31)));
        asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(m) : "memory");
      }
    }
  } else if constexpr (R == 2) {
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t k = tid; k < n; k += stride) {
      const uint64_t h = key_hash(seed, k);
      uint32_t* p = buf + __umul64hi(h, nb) * 8;
#pragma unroll
      for (int w = 0; w < 8; ++w)
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p + w), "r"(1u << ((h >> (4 * w)) & 31)) : "memory");
    }
  }
}

template <typename K>
float time_it(K launch) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  launch();
  float best = 1e30f;
  for (int i = 0; i < 3; ++i) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t n = 1ull << 28;
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4096));
  const uint64_t sizes_mib[] = {1, 64, 128, 1024, 4096};
  for (uint64_t mib : sizes_mib) {
    uint32_t* buf;
    const uint64_t bytes = mib << 20, nb = bytes / 32;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    const int grid = sms * 4;
#define RD(F, name)                                                                              \
  {                                                                                              \
    float ms = time_it([&] { read_kernel<F><<<grid, 256>>>(buf, nb, n, 7 + F, sink); });        \
    printf("read  %-28s buf=%6llu MiB  %8.2f G/s\n", name, (unsigned long long)mib, n / ms / 1e6); \
  }
    RD(0, "nc.noalloc.evict_last.v8");
    RD(1, "nc.v8");
    RD(2, "plain.v8");
    RD(3, "cg.v8");
    RD(4, "cs.v8");
    RD(5, "cv.v8");
    RD(6, "nc.noalloc 2x v4");
    RD(7, "nc.noalloc.evict_first.v8");
    RD(8, "nc.noalloc.u32 (4 B)");
    RD(9, "relaxed.gpu.v8");
#define RE(R, name)                                                                              \
  {                                                                                              \
    float ms = time_it([&] { red_kernel<R><<<grid, 256>>>(buf, nb, n, 11 + R); });              \
    printf("red   %-28s buf=%6llu MiB  %8.2f G/s\n", name, (unsigned long long)mib, n / ms / 1e6); \
  }
    RE(0, "lane8 red.b32");
    RE(1, "lane4 red.b64");
    RE(2, "thread 8x red.b32");
    RE(3, "lane8 atom.or.b32");
    RE(4, "lane8 test+red.b32");
    fflush(stdout);
    CK(cudaFree(buf));
  }
  return 0;
}
