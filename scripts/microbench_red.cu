// microbench_red.cu — what bounds the L2-resident insert (config 2: 1M keys
// into a 1 MiB filter)? Design evidence for insert_wide_kernel; not part of
// the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/microbench_red scripts/microbench_red.cu
//   scripts/bin/microbench_red
//
// Every variant does 4 lanes per key, one red.global.or.b64 per lane pair (as
// insert_wide_kernel). Variants:
//   regs     : keys from splitmix64 in registers (no hash stream)
//   stream   : keys loaded from a device array (the real kernel's input)
//   hint     : red with an L2::evict_last cache hint (as the product) or none
//   grid     : "once" = one warp step per warp, grid covering the batch once
//              (the product's WIDE launch); "persist" = k CTAs per SM looping
// Before each timed rep a 256 MiB buffer is written and another read, so
// the key array and the filter start cold, as in bench.py.
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

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int kHint>  // 0 none, 1 evict_last, 2 evict_first
__device__ __forceinline__ void red64(uint64_t* p, uint64_t v, uint64_t pol) {
  if constexpr (kHint == 0)
    asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ uint64_t pair_mask(uint32_t low, int pair) {
  const uint32_t s[8] = {0x44974d91u, 0x47b6137bu, 0xa2b7289du, 0x8824ad5bu,
                         0x2df1424bu, 0x705495c7u, 0x5c6bfb31u, 0x9efc4947u};
  uint32_t lo = s[0], hi = s[1];
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (pair == k) {
      lo = s[2 * k];
      hi = s[2 * k + 1];
    }
  return (uint64_t(1u << ((hi * low) >> 27)) << 32) | (1u << ((lo * low) >> 27));
}

// kSrc: 0 = keys in registers, 1 = keys from `keys`
template <int kSrc, int kHint, int kT>
__global__ void __launch_bounds__(256, 4) ins_kernel(uint32_t* __restrict__ blocks, uint64_t nb,
                                                     const uint64_t* __restrict__ keys, uint64_t n) {
  const int lane = threadIdx.x & 31, sub = lane >> 2, pair = lane & 3;
  const uint64_t pol = kHint == 2 ? pol_first() : pol_last();
  const uint64_t spol = pol_first();
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t nsteps = (n + 32 * kT - 1) / (32 * kT);
  for (uint64_t t = warp; t < nsteps; t += nwarps) {
    const uint64_t base = t * 32 * kT;
    uint64_t h[kT];
#pragma unroll
    for (int j = 0; j < kT; ++j) {
      const uint64_t idx = base + j * 32 + lane;
      if constexpr (kSrc == 0) h[j] = mix(0x1234 + (idx + 1) * 0x9e3779b97f4a7c15ull);
      else h[j] = idx < n ? ld_stream(keys + idx, spol) : 0;
    }
#pragma unroll
    for (int j = 0; j < kT; ++j) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int k = r * 8 + sub;
        const uint64_t hk = __shfl_sync(0xffffffffu, h[j], k);
        if (base + j * 32 + k < n) {
          uint64_t* p = reinterpret_cast<uint64_t*>(blocks + __umul64hi(hk, nb) * 8) + pair;
          red64<kHint>(p, pair_mask(uint32_t(hk), pair), pol);
        }
      }
    }
  }
}

struct Bufs {
  uint32_t* filter;
  uint64_t* keys;
  uint8_t* flush_w;
  int* flush_r;
  int* sink;
};

__global__ void sum_kernel(const int* __restrict__ p, uint64_t n, int* out) {
  int acc = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    acc += p[i];
  if (acc == 0x7fffffff) *out = acc;
}

__global__ void empty_kernel() {}

template <typename L>
void run(const char* name, Bufs& b, uint64_t nb, uint64_t n, int sms, L launch, bool cold = true) {
  const uint64_t flush = 256ull << 20;
  std::vector<float> t;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int rep = 0; rep < 23; ++rep) {
    CK(cudaMemsetAsync(b.filter, 0, nb * 32));
    if (cold) {
      CK(cudaMemsetAsync(b.flush_w, rep, flush));
      sum_kernel<<<sms * 4, 256>>>(b.flush_r, flush / 4, b.sink);
    }
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep >= 3) t.push_back(ms);
  }
  CK(cudaGetLastError());
  std::sort(t.begin(), t.end());
  const float med = t[t.size() / 2];
  printf("%-44s n=%10llu  %8.2f us  %7.1f Gkeys/s\n", name, (unsigned long long)n, med * 1e3, n / med / 1e6);
  fflush(stdout);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t nb = 32768;  // config 2's 1 MiB filter
  const uint64_t nmax = 1ull << 26;
  Bufs b;
  CK(cudaMalloc(&b.filter, nb * 32));
  CK(cudaMalloc(&b.keys, nmax * 8));
  CK(cudaMalloc(&b.flush_w, 256ull << 20));
  CK(cudaMalloc(&b.flush_r, 256ull << 20));
  CK(cudaMalloc(&b.sink, 64));
  CK(cudaMemset(b.flush_r, 0, 256ull << 20));
  std::vector<uint64_t> h(nmax);
  for (uint64_t i = 0; i < nmax; ++i) h[i] = mix(3 + (i + 1) * 0x9e3779b97f4a7c15ull);
  CK(cudaMemcpy(b.keys, h.data(), nmax * 8, cudaMemcpyHostToDevice));
  run("empty kernel (launch + event overhead)", b, nb, 0, sms, [] { empty_kernel<<<1, 32>>>(); });
  run("2 empty kernels", b, nb, 0, sms, [] { empty_kernel<<<1, 32>>>(); empty_kernel<<<1, 32>>>(); });
  run("empty kernel, 1184 CTAs", b, nb, 0, sms, [=] { empty_kernel<<<sms * 8, 256>>>(); });
  run("empty kernel, GPU idle before (no flush)", b, nb, 0, sms, [] { empty_kernel<<<1, 32>>>(); }, false);
  {
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const uint64_t n = 1000000;
    const unsigned grid = unsigned((n + 1023) / 1024);
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeGlobal));
    ins_kernel<1, 0, 4><<<grid, 256, 0, cs>>>(b.filter, nb, b.keys, n);
    CK(cudaStreamEndCapture(cs, &gr));
    CK(cudaGraphInstantiate(&ge, gr, 0));
    run("stream hint=none once T=4, CUDA graph", b, nb, n, sms, [=] { CK(cudaGraphLaunch(ge, 0)); });
  }
  for (int per_sm : {2, 3, 4, 6, 8, 12, 16}) {
    const uint64_t n = 1000000;
    char name[64];
    snprintf(name, sizeof name, "stream hint=none persist %d/SM T=2", per_sm);
    run(name, b, nb, n, sms, [=] { ins_kernel<1, 0, 2><<<sms * per_sm, 256>>>(b.filter, nb, b.keys, n); });
    snprintf(name, sizeof name, "stream hint=none persist %d/SM T=1", per_sm);
    run(name, b, nb, n, sms, [=] { ins_kernel<1, 0, 1><<<sms * per_sm, 256>>>(b.filter, nb, b.keys, n); });
  }
  run("stream hint=none once T=1", b, nb, 1000000, sms,
      [=] { ins_kernel<1, 0, 1><<<unsigned((1000000 + 255) / 256), 256>>>(b.filter, nb, b.keys, 1000000); });
  for (uint64_t n : {uint64_t{1000000}, uint64_t{2000000}, uint64_t{4000000}}) {
    const unsigned grid = unsigned((n + 1023) / 1024);
    run("regs   hint=none  once T=4 WARM filter", b, nb, n, sms,
        [=] { ins_kernel<0, 0, 4><<<grid, 256>>>(b.filter, nb, b.keys, n); }, false);
    run("regs   hint=none  once T=4", b, nb, n, sms,
        [=] { ins_kernel<0, 0, 4><<<grid, 256>>>(b.filter, nb, b.keys, n); });
    run("stream hint=none  once T=4 WARM", b, nb, n, sms,
        [=] { ins_kernel<1, 0, 4><<<grid, 256>>>(b.filter, nb, b.keys, n); }, false);
  }
  for (uint64_t n : {uint64_t{1000000}, uint64_t{1} << 26}) {
    auto once = [&](auto kern, int kt) {
      const unsigned grid = unsigned((n + 256 * kt - 1) / (256 * kt));
      return [=] { kern<<<grid, 256>>>(b.filter, nb, b.keys, n); };
    };
    auto persist = [&](auto kern, int per_sm) {
      return [=] { kern<<<sms * per_sm, 256>>>(b.filter, nb, b.keys, n); };
    };
    run("regs   hint=last  once T=4", b, nb, n, sms, once(ins_kernel<0, 1, 4>, 4));
    run("regs   hint=none  once T=4", b, nb, n, sms, once(ins_kernel<0, 0, 4>, 4));
    run("stream hint=last  once T=4 (product WIDE)", b, nb, n, sms, once(ins_kernel<1, 1, 4>, 4));
    run("stream hint=none  once T=4", b, nb, n, sms, once(ins_kernel<1, 0, 4>, 4));
    run("stream hint=first once T=4", b, nb, n, sms, once(ins_kernel<1, 2, 4>, 4));
    run("stream hint=none  once T=2", b, nb, n, sms, once(ins_kernel<1, 0, 2>, 2));
    run("stream hint=none  once T=8", b, nb, n, sms, once(ins_kernel<1, 0, 8>, 8));
    run("stream hint=none  persist 4/SM T=4", b, nb, n, sms, persist(ins_kernel<1, 0, 4>, 4));
    run("stream hint=none  persist 8/SM T=2", b, nb, n, sms, persist(ins_kernel<1, 0, 2>, 8));
    run("stream hint=last  persist 4/SM T=4", b, nb, n, sms, persist(ins_kernel<1, 1, 4>, 4));
  }
  return 0;
}
