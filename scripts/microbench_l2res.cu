// microbench_l2res.cu — does a filter slice stay L2-resident while keys stream
// past it? A stripped-down blocked sweep: region r of a 1 GiB "filter" is
// probed by the keys of the contiguous key range r (CTAs in blockIdx order
// walk regions 0..R-1, as segment_kernel walks buckets). Variants change the
// L2 policy of the three streams (keys in, probe, answer out), the MLP per
// thread and the region size; one launch per variant, CUDA-event timed.
// Run under ncu --metrics dram__bytes_read.sum to see the filter refetches.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o scripts/bin/microbench_l2res scripts/microbench_l2res.cu
//   scripts/bin/microbench_l2res [variant_mask]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void gen_keys(uint64_t* k, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    k[i] = fmix(0x1234 + (i + 1) * 0x9e3779b97f4a7c15ull);
}

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// flags
enum : int {
  kProbeLast = 1,     // probe loads with an evict_last policy
  kOutFirst = 2,      // answer stores with an evict_first policy
  kDiscard = 4,       // discard.global.L2 the key lines after they are consumed
  kKeysNormal = 8,    // keys loaded without the evict_first hint
  kOutNone = 16,      // no answer stores (reduced to a per-thread xor)
  kChunked = 32,      // keys in the blocked path's chunk-local layout: region r's keys are 128-key
                      // runs at chunk*4096 + r*128 (32 KB stride)
  kChunkedPad = 64,   // the same with a 4128-key (33 KB) chunk stride
  kAhead1 = 128,      // each CTA bulk-prefetches its share of region r+1 into L2 first
  kAhead2 = 256,      // ... of region r+2
};

// CTA g of `groups` prefetches its share of region rr (if it exists)
__device__ __forceinline__ void prefetch_share(const uint32_t* filt, uint64_t region_blocks, uint64_t regions,
                                               uint64_t rr, uint32_t g, uint32_t groups) {
  if (rr >= regions || threadIdx.x != 0) return;
  const uint64_t bytes = region_blocks * 32, share = (bytes / groups) & ~15ull;
  const char* p = reinterpret_cast<const char*>(filt + rr * region_blocks * 8) + g * share;
  if (share) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)share) : "memory");
}

template <int F>
__device__ __forceinline__ uint64_t key_addr(uint64_t i, uint64_t r, uint64_t per_region) {
  if (!(F & (kChunked | kChunkedPad))) return i;
  const uint64_t li = i - r * per_region, ch = li >> 7, off = li & 127;
  return ch * ((F & kChunkedPad) ? 4128 : 4096) + r * 128 + off;
}

template <int F, int U>
__global__ void __launch_bounds__(256, 8) sweep(const uint32_t* __restrict__ filt, uint64_t region_blocks,
                                                 const uint64_t* __restrict__ keys, uint64_t per_region,
                                                 uint32_t groups, uint8_t* __restrict__ out, uint32_t* sink) {
  const uint32_t r = blockIdx.x / groups, g = blockIdx.x % groups;
  const uint64_t per_cta = (per_region + groups - 1) / groups;
  const uint64_t k0 = r * per_region + g * per_cta;
  uint64_t k1 = k0 + per_cta;
  if (k1 > (r + 1) * per_region) k1 = (r + 1) * per_region;
  const uint32_t* base = filt + r * region_blocks * 8;
  const uint64_t pf = pol_first(), pl = pol_last();
  uint32_t acc = 0;
  if (F & kAhead1) prefetch_share(filt, region_blocks, (1ull << 30) / (region_blocks * 32), r + 1, g, groups);
  if (F & kAhead2) prefetch_share(filt, region_blocks, (1ull << 30) / (region_blocks * 32), r + 2, g, groups);
  for (uint64_t i0 = k0 + threadIdx.x; i0 < k1; i0 += 256 * U) {
    uint64_t h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * 256;
      if (i < k1) {
        const uint64_t ka = key_addr<F>(i, r, per_region);
        if (F & kKeysNormal)
          asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(h[u]) : "l"(keys + ka));
        else
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(h[u]) : "l"(keys + ka), "l"(pf));
      } else {
        h[u] = 0;
      }
    }
    uint32_t w[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t* p = base + __umul64hi(h[u], region_blocks) * 8;
      if (F & kProbeLast)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=r"(w[u][0]), "=r"(w[u][1]), "=r"(w[u][2]), "=r"(w[u][3]), "=r"(w[u][4]), "=r"(w[u][5]),
                       "=r"(w[u][6]), "=r"(w[u][7])
                     : "l"(p), "l"(pl));
      else
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[u][0]), "=r"(w[u][1]), "=r"(w[u][2]), "=r"(w[u][3]), "=r"(w[u][4]), "=r"(w[u][5]),
                       "=r"(w[u][6]), "=r"(w[u][7])
                     : "l"(p));
    }
    if (F & kDiscard) {
      // the warp's 32 keys of step u are 256 B = two 128-B lines; lanes 0 and
      // 16 discard them (after the loads above consumed them)
      const uint32_t lane = threadIdx.x & 31;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = i0 + u * 256;
        if ((lane & 15) == 0 && i + 15 < k1 && ((reinterpret_cast<uintptr_t>(keys + i) & 127) == 0))
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(keys + i) : "memory");
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t low = (uint32_t)h[u];
      uint32_t miss = 0;
#pragma unroll
      for (int l = 0; l < 8; ++l) miss |= (1u << ((0x44974d91u * (l + 1) * low) >> 27)) & ~w[u][l];
      const uint64_t i = i0 + u * 256;
      if (F & kOutNone) {
        acc ^= miss;
      } else if (i < k1) {
        if (F & kOutFirst)
          asm volatile("st.global.L1::no_allocate.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(out + i), "r"(miss == 0 ? 1u : 0u), "l"(pf)
                       : "memory");
        else
          asm volatile("st.global.L1::no_allocate.u8 [%0], %1;" ::"l"(out + key_addr<F>(i, r, per_region)), "r"(miss == 0 ? 1u : 0u) : "memory");
      }
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}


// Insert sweep over the same region layout. M: 0 = 4 threads/key, one
// red.or.b64 per lane pair; 1 = same with test-before-set (load the pair,
// red only missing bits); 2 = 8 threads/key, red.or.b32 per lane; 3 = one
// thread/key issuing the 4 pair reds.
template <int M>
__global__ void __launch_bounds__(256, 8) isweep(uint32_t* __restrict__ filt, uint64_t region_blocks,
                                                  const uint64_t* __restrict__ keys, uint64_t per_region,
                                                  uint32_t groups) {
  const uint32_t r = blockIdx.x / groups, g = blockIdx.x % groups;
  const uint64_t per_cta = (per_region + groups - 1) / groups;
  const uint64_t k0 = r * per_region + g * per_cta;
  uint64_t k1 = k0 + per_cta;
  if (k1 > (r + 1) * per_region) k1 = (r + 1) * per_region;
  uint32_t* base = filt + r * region_blocks * 8;
  const uint64_t pf = pol_first(), pl = pol_last();
  constexpr int TPK = M == 2 ? 8 : (M == 3 ? 1 : 4);
  const uint32_t sub = threadIdx.x % TPK;
  if (M == 8) prefetch_share(filt, region_blocks, (1ull << 30) / (region_blocks * 32), r + 1, g, groups);
  if (M == 9) prefetch_share(filt, region_blocks, (1ull << 30) / (region_blocks * 32), r + 2, g, groups);
  if (M == 6 || M == 7) {
    // prefetch this CTA's share of the region into L2 first (128-B lines)
    const uint64_t bytes = region_blocks * 32, share = (bytes + groups - 1) / groups;
    const uint64_t b0 = g * share, b1 = b0 + share < bytes ? b0 + share : bytes;
    const char* rb = reinterpret_cast<const char*>(base);
    if (M == 6) {
      if (threadIdx.x == 0 && b1 > b0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rb + b0), "r"((uint32_t)((b1 - b0) & ~15ull)) : "memory");
    } else {
      uint32_t acc = 0;
      for (uint64_t o = b0 + threadIdx.x * 16; o + 16 <= b1; o += 256 * 16) {
        uint32_t a, b2, c, d;
        asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(a), "=r"(b2), "=r"(c), "=r"(d) : "l"(rb + o), "l"(pl));
        acc ^= a;
      }
      if (acc == 0x9abcdef1u) filt[0] = acc;
    }
  }
  for (uint64_t i = k0 + threadIdx.x / TPK; i < k1; i += 256 / TPK) {
    uint64_t h;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(h) : "l"(keys + i), "l"(pf));
    const uint32_t low = (uint32_t)h;
    uint32_t* b = base + __umul64hi(h, region_blocks) * 8;
    if (M == 2) {
      const uint32_t m = 1u << ((0x44974d91u * (sub + 1) * low) >> 27);
      asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(b + sub), "r"(m) : "memory");
    } else if (M == 3) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t m = ((uint64_t)(1u << ((0x44974d91u * (2 * q + 2) * low) >> 27)) << 32) |
                           (1u << ((0x44974d91u * (2 * q + 1) * low) >> 27));
        asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(reinterpret_cast<uint64_t*>(b) + q), "l"(m) : "memory");
      }
    } else {
      const uint64_t m = ((uint64_t)(1u << ((0x44974d91u * (2 * sub + 2) * low) >> 27)) << 32) |
                         (1u << ((0x44974d91u * (2 * sub + 1) * low) >> 27));
      uint64_t* p = reinterpret_cast<uint64_t*>(b) + sub;
      bool need = true;
      if (M == 1) {
        uint64_t cur;
        asm volatile("ld.global.u64 %0, [%1];" : "=l"(cur) : "l"(p));
        need = (m & ~cur) != 0;
      }
      if (M == 5 || M == 8 || M == 9) {
        uint64_t cur;
        asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(cur) : "l"(p), "l"(pl));
        need = (m & ~cur) != 0;
      }
      if (need) {
        if (M >= 4)
          asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(m), "l"(pl) : "memory");
        else
          asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(m) : "memory");
      }
    }
  }
}

template <int M>
float irun(uint32_t* filt, uint64_t filter_blocks, uint64_t region_blocks, const uint64_t* keys, uint64_t n,
           const char* name) {
  const uint64_t regions = filter_blocks / region_blocks;
  const uint64_t per_region = n / regions;
  const uint32_t groups = (uint32_t)((per_region + 8191) / 8192);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaMemset(filt, 0, filter_blocks * 32));
  isweep<M><<<(unsigned)(regions * groups), 256>>>(filt, region_blocks, keys, per_region, groups);
  CK(cudaMemset(filt, 0, filter_blocks * 32));
  CK(cudaEventRecord(a));
  isweep<M><<<(unsigned)(regions * groups), 256>>>(filt, region_blocks, keys, per_region, groups);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("insert %-27s region=%5.0f MiB  n=%llu %8.3f ms  %7.1f G keys/s\n", name, region_blocks * 32.0 / (1 << 20),
         (unsigned long long)n, ms, n / (ms * 1e-3) / 1e9);
  fflush(stdout);
  return ms;
}


// Persistent sweep: grid = resident CTAs; every CTA walks the regions in
// order and takes its share of each region's keys, so all CTAs work on the
// same region (+- drift). SYNC: before region r+2, wait until every CTA has
// finished region r (global counters, spin). INS: insert (test+red el) or lookup.
template <bool INS, bool SYNC, int U>
__global__ void __launch_bounds__(256, 4) psweep(uint32_t* __restrict__ filt, uint64_t region_blocks, uint64_t regions,
                                                  const uint64_t* __restrict__ keys, uint64_t per_region,
                                                  uint8_t* __restrict__ out, unsigned* __restrict__ done) {
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t share = (per_region + gridDim.x - 1) / gridDim.x;
  for (uint64_t r = 0; r < regions; ++r) {
    if (SYNC && r >= 2) {
      if (threadIdx.x == 0) {
        volatile unsigned* d = done + r - 2;
        while (*d < gridDim.x) __nanosleep(100);
      }
      __syncthreads();
    }
    uint32_t* base = filt + r * region_blocks * 8;
    const uint64_t k0 = r * per_region + blockIdx.x * share;
    uint64_t k1 = k0 + share;
    if (k1 > (r + 1) * per_region) k1 = (r + 1) * per_region;
    if (INS) {
      const uint32_t sub = threadIdx.x & 3;
      for (uint64_t i0 = k0 + threadIdx.x / 4; i0 < k1; i0 += 64 * U) {
        uint64_t h[U], cur[U], m[U];
        uint64_t* p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + u * 64;
          h[u] = 0;
          if (i < k1) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(h[u]) : "l"(keys + i), "l"(pf));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t low = (uint32_t)h[u];
          p[u] = reinterpret_cast<uint64_t*>(base + __umul64hi(h[u], region_blocks) * 8) + sub;
          m[u] = i0 + u * 64 < k1 ? ((uint64_t)(1u << ((0x44974d91u * (2 * sub + 2) * low) >> 27)) << 32) |
                                        (1u << ((0x44974d91u * (2 * sub + 1) * low) >> 27)) : 0;
          asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(cur[u]) : "l"(p[u]), "l"(pl));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (m[u] & ~cur[u])
            asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p[u]), "l"(m[u]), "l"(pl) : "memory");
      }
    } else {
      for (uint64_t i0 = k0 + threadIdx.x; i0 < k1; i0 += 256 * U) {
        uint64_t h[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + u * 256;
          h[u] = 0;
          if (i < k1) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(h[u]) : "l"(keys + i), "l"(pf));
        }
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t* q = base + __umul64hi(h[u], region_blocks) * 8;
          asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(w[u][0]), "=r"(w[u][1]), "=r"(w[u][2]), "=r"(w[u][3]), "=r"(w[u][4]), "=r"(w[u][5]),
                         "=r"(w[u][6]), "=r"(w[u][7])
                       : "l"(q));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t low = (uint32_t)h[u];
          uint32_t miss = 0;
#pragma unroll
          for (int l = 0; l < 8; ++l) miss |= (1u << ((0x44974d91u * (l + 1) * low) >> 27)) & ~w[u][l];
          const uint64_t i = i0 + u * 256;
          if (i < k1) asm volatile("st.global.L1::no_allocate.u8 [%0], %1;" ::"l"(out + i), "r"(miss == 0 ? 1u : 0u) : "memory");
        }
      }
    }
    if (SYNC) {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(done + r, 1u);
      }
    }
  }
}

template <bool INS, bool SYNC, int U>
float prun(uint32_t* filt, uint64_t filter_blocks, uint64_t region_blocks, const uint64_t* keys, uint64_t n,
           uint8_t* out, unsigned* done, int ctas_per_sm, const char* name) {
  const uint64_t regions = filter_blocks / region_blocks;
  const uint64_t per_region = n / regions;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const unsigned grid = sms * ctas_per_sm;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float ms = 0;
  for (int it = 0; it < 2; ++it) {
    if (INS) CK(cudaMemset(filt, 0, filter_blocks * 32));
    CK(cudaMemset(done, 0, 4096));
    CK(cudaEventRecord(a));
    psweep<INS, SYNC, U><<<grid, 256>>>(filt, region_blocks, regions, keys, per_region, out, done);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
  }
  printf("persistent %s %-6s sync=%d U=%d ctas/sm=%d region=%5.0f MiB n=%llu %8.3f ms %7.1f G keys/s\n",
         INS ? "insert" : "lookup", name, (int)SYNC, U, ctas_per_sm, region_blocks * 32.0 / (1 << 20),
         (unsigned long long)n, ms, n / (ms * 1e-3) / 1e9);
  fflush(stdout);
  return ms;
}

template <int F, int U>
float run(const uint32_t* filt, uint64_t filter_blocks, uint64_t region_blocks, const uint64_t* keys, uint64_t n,
          uint8_t* out, uint32_t* sink, const char* name) {
  const uint64_t regions = filter_blocks / region_blocks;
  const uint64_t per_region = n / regions;
  const uint32_t groups = (uint32_t)((per_region + 8191) / 8192);  // ~8192 keys per CTA, as segment_kernel
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  // one warm-up launch, then the timed one
  sweep<F, U><<<(unsigned)(regions * groups), 256>>>(filt, region_blocks, keys, per_region, groups, out, sink);
  CK(cudaEventRecord(a));
  sweep<F, U><<<(unsigned)(regions * groups), 256>>>(filt, region_blocks, keys, per_region, groups, out, sink);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("%-34s region=%5.0f MiB U=%d  %8.3f ms  %7.1f G probes/s\n", name, region_blocks * 32.0 / (1 << 20), U, ms,
         n / (ms * 1e-3) / 1e9);
  fflush(stdout);
  return ms;
}

int main(int argc, char** argv) {
  const unsigned mask = argc > 1 ? (unsigned)strtoul(argv[1], nullptr, 0) : ~0u;
  const uint64_t filter_blocks = 1ull << 25;  // 1 GiB
  const uint64_t n = 1ull << 28;
  uint32_t* filt;
  uint64_t* keys;
  uint8_t* out;
  uint32_t* sink;
  CK(cudaMalloc(&filt, filter_blocks * 32));
  CK(cudaMemset(filt, 0x5a, filter_blocks * 32));
  CK(cudaMalloc(&keys, n * 8 + (n / 4096) * 32 * 8));
  CK(cudaMalloc(&out, n + (n / 4096) * 32));
  CK(cudaMalloc(&sink, 64));
  gen_keys<<<1184, 256>>>(keys, n + (n / 4096) * 32);
  CK(cudaDeviceSynchronize());
  const uint64_t r32 = (32ull << 20) / 32, r16 = (16ull << 20) / 32, r64 = (64ull << 20) / 32, r8 = (8ull << 20) / 32;
  if (mask & 1) run<0, 1>(filt, filter_blocks, r32, keys, n, out, sink, "baseline (keys ef, probe normal)");
  if (mask & 2) run<kProbeLast, 1>(filt, filter_blocks, r32, keys, n, out, sink, "probe evict_last");
  if (mask & 4) run<kOutFirst, 1>(filt, filter_blocks, r32, keys, n, out, sink, "out evict_first");
  if (mask & 8) run<kDiscard, 1>(filt, filter_blocks, r32, keys, n, out, sink, "discard keys");
  if (mask & 16) run<kProbeLast | kOutFirst | kDiscard, 1>(filt, filter_blocks, r32, keys, n, out, sink, "all three");
  if (mask & 32) run<kOutNone, 1>(filt, filter_blocks, r32, keys, n, out, sink, "no answer stores");
  if (mask & 64) run<kKeysNormal, 1>(filt, filter_blocks, r32, keys, n, out, sink, "keys normal policy");
  if (mask & 128) run<0, 2>(filt, filter_blocks, r32, keys, n, out, sink, "baseline");
  if (mask & 256) run<0, 4>(filt, filter_blocks, r32, keys, n, out, sink, "baseline");
  if (mask & 512) run<kProbeLast | kOutFirst | kDiscard, 4>(filt, filter_blocks, r32, keys, n, out, sink, "all three");
  if (mask & 1024) run<0, 1>(filt, filter_blocks, r16, keys, n, out, sink, "baseline");
  if (mask & 2048) run<0, 1>(filt, filter_blocks, r64, keys, n, out, sink, "baseline");
  if (mask & 4096) run<0, 1>(filt, filter_blocks, r8, keys, n, out, sink, "baseline");
  if (mask & 8192) run<kProbeLast | kOutFirst | kDiscard, 1>(filt, filter_blocks, r16, keys, n, out, sink, "all three");
  if (mask & 16384) run<kProbeLast | kOutFirst | kDiscard, 1>(filt, filter_blocks, r64, keys, n, out, sink, "all three");
  if (mask & 32768) run<kOutNone, 4>(filt, filter_blocks, r32, keys, n, out, sink, "no answer stores");
  if (mask & (1u << 14)) {  // prefetch-ahead of the next region(s)
    run<0, 1>(filt, filter_blocks, r16, keys, n, out, sink, "16 MiB, no prefetch");
    run<kAhead1, 1>(filt, filter_blocks, r16, keys, n, out, sink, "16 MiB, prefetch r+1");
    run<kAhead2, 1>(filt, filter_blocks, r16, keys, n, out, sink, "16 MiB, prefetch r+2");
    run<kAhead1, 1>(filt, filter_blocks, r8, keys, n, out, sink, "8 MiB, prefetch r+1");
    run<kAhead1, 1>(filt, filter_blocks, r32, keys, n, out, sink, "32 MiB, prefetch r+1");
    const uint64_t ni = 1ull << 26;
    irun<5>(filt, filter_blocks, r16, keys, ni, "test+red el 16 MiB");
    irun<8>(filt, filter_blocks, r16, keys, ni, "test+red el 16 MiB, pf r+1");
    irun<9>(filt, filter_blocks, r16, keys, ni, "test+red el 16 MiB, pf r+2");
    irun<8>(filt, filter_blocks, r8, keys, ni, "test+red el 8 MiB, pf r+1");
    irun<8>(filt, filter_blocks, r32, keys, ni, "test+red el 32 MiB, pf r+1");
  }
  if (mask & (1u << 31)) {
    run<0, 1>(filt, filter_blocks, r32, keys, n, out, sink, "flat keys");
    run<kChunked, 1>(filt, filter_blocks, r32, keys, n, out, sink, "chunk-local keys, 32 KB stride");
    run<kChunkedPad, 1>(filt, filter_blocks, r32, keys, n, out, sink, "chunk-local keys, 33 KB stride");
    run<kChunked | kOutNone, 1>(filt, filter_blocks, r32, keys, n, out, sink, "chunk-local, no answers");
    run<kChunked, 1>(filt, filter_blocks, r16, keys, n, out, sink, "chunk-local keys, 32 KB stride");
  }
  const uint64_t ni = 1ull << 26;  // one config-4 insert chunk
  if (mask & (1u << 16)) irun<0>(filt, filter_blocks, r32, keys, ni, "4 thr/key red.b64");
  if (mask & (1u << 17)) irun<1>(filt, filter_blocks, r32, keys, ni, "4 thr/key test+red.b64");
  if (mask & (1u << 18)) irun<2>(filt, filter_blocks, r32, keys, ni, "8 thr/key red.b32");
  if (mask & (1u << 19)) irun<3>(filt, filter_blocks, r32, keys, ni, "1 thr/key 4x red.b64");
  if (mask & (1u << 20)) irun<0>(filt, filter_blocks, r16, keys, ni, "4 thr/key red.b64");
  if (mask & (1u << 21)) irun<0>(filt, filter_blocks, r8, keys, ni, "4 thr/key red.b64");
  if (mask & (1u << 22)) irun<0>(filt, filter_blocks, r32, keys, n, "4 thr/key red.b64");
  if (mask & (1u << 23)) irun<1>(filt, filter_blocks, r16, keys, ni, "4 thr/key test+red.b64");
  if (mask & (1u << 24)) irun<4>(filt, filter_blocks, r32, keys, ni, "red.b64 evict_last");
  if (mask & (1u << 25)) irun<5>(filt, filter_blocks, r32, keys, ni, "test+red evict_last");
  if (mask & (1u << 26)) irun<6>(filt, filter_blocks, r32, keys, ni, "bulk prefetch + red el");
  if (mask & (1u << 27)) irun<7>(filt, filter_blocks, r32, keys, ni, "ld prefetch + red el");
  if (mask & (1u << 28)) {
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 128));
    irun<0>(filt, filter_blocks, r32, keys, ni, "red.b64 fetch gran 128");
    irun<4>(filt, filter_blocks, r32, keys, ni, "red.b64 el fetch gran 128");
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32));
    irun<0>(filt, filter_blocks, r32, keys, ni, "red.b64 fetch gran 32");
  }
  if (mask & (1u << 29)) irun<6>(filt, filter_blocks, r16, keys, ni, "bulk prefetch + red el");
  if (mask & (1u << 30)) {
    unsigned* done;
    CK(cudaMalloc(&done, 4096));
    prun<true, false, 1>(filt, filter_blocks, r32, keys, ni, out, done, 4, "");
    prun<true, true, 1>(filt, filter_blocks, r32, keys, ni, out, done, 4, "");
    prun<true, true, 2>(filt, filter_blocks, r32, keys, ni, out, done, 4, "");
    prun<true, true, 4>(filt, filter_blocks, r32, keys, ni, out, done, 4, "");
    prun<true, true, 2>(filt, filter_blocks, r16, keys, ni, out, done, 4, "");
    prun<true, true, 2>(filt, filter_blocks, r32, keys, ni, out, done, 8, "");
    prun<true, true, 2>(filt, filter_blocks, r32, keys, n, out, done, 4, "");
    prun<false, false, 1>(filt, filter_blocks, r32, keys, n, out, done, 4, "");
    prun<false, true, 1>(filt, filter_blocks, r32, keys, n, out, done, 4, "");
    prun<false, true, 2>(filt, filter_blocks, r32, keys, n, out, done, 4, "");
    prun<false, true, 4>(filt, filter_blocks, r32, keys, n, out, done, 4, "");
    prun<false, true, 2>(filt, filter_blocks, r32, keys, n, out, done, 8, "");
    prun<false, true, 2>(filt, filter_blocks, r16, keys, n, out, done, 4, "");
    prun<false, true, 2>(filt, filter_blocks, r64, keys, n, out, done, 4, "");
    prun<false, true, 2>(filt, filter_blocks, r32, keys, n / 2, out, done, 4, "");
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
