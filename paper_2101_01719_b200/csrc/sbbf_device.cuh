// sbbf_device.cuh — device-side SBBF semantics and memory primitives (sm_100a).
//
// Semantics follow the reference core exactly (paths relative to
// /root/reference/proj/):
//   kLaneSeeds   core/include/sbbf/filter.hpp:18-21
//   block_index  core/src/filter.cpp:15-29,125-127  -> __umul64hi
//   make_mask    core/src/filter.cpp:129-138        -> IMAD + SHF + SHL per lane
//   find         core/src/filter.cpp:38-46,71-77    -> (~block & mask) == 0
#pragma once

#include <cstdint>
#include <cstdio>

// Device-side bounds checks for the debug build (`make debug`:
// libsbbf_gpu_debug.so, -DSBBF_DEBUG). compute-sanitizer is unavailable on
// the GPU pool, so the test suite runs once against this build instead; a
// failed check prints its location and traps. Compiled out otherwise.
#ifdef SBBF_DEBUG
#define SBBF_DCHECK(c)                                                               \
  do {                                                                               \
    if (!(c)) {                                                                      \
      printf("SBBF_DCHECK failed: %s at %s:%d\n", #c, __FILE__, __LINE__);           \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define SBBF_DCHECK(c) ((void)0)
#endif

namespace sbbf {
namespace dev {

constexpr int kLanes = 8;
constexpr uint32_t kSeed0 = 0x44974d91u, kSeed1 = 0x47b6137bu, kSeed2 = 0xa2b7289du,
                   kSeed3 = 0x8824ad5bu, kSeed4 = 0x2df1424bu, kSeed5 = 0x705495c7u,
                   kSeed6 = 0x5c6bfb31u, kSeed7 = 0x9efc4947u;

__host__ __device__ constexpr uint32_t lane_seed(int i) {
  return i == 0   ? kSeed0
         : i == 1 ? kSeed1
         : i == 2 ? kSeed2
         : i == 3 ? kSeed3
         : i == 4 ? kSeed4
         : i == 5 ? kSeed5
         : i == 6 ? kSeed6
                  : kSeed7;
}

// Lane seed selected at run time (lane-parallel kernels): a byte-permute free
// select from immediates, no local-memory array.
__device__ __forceinline__ uint32_t lane_seed_rt(int i) {
  uint32_t s = kSeed0;
  s = (i == 1) ? kSeed1 : s;
  s = (i == 2) ? kSeed2 : s;
  s = (i == 3) ? kSeed3 : s;
  s = (i == 4) ? kSeed4 : s;
  s = (i == 5) ? kSeed5 : s;
  s = (i == 6) ? kSeed6 : s;
  s = (i == 7) ? kSeed7 : s;
  return s;
}

__device__ __forceinline__ uint64_t block_index(uint64_t hash, uint64_t num_buckets) {
  return __umul64hi(hash, num_buckets);
}

__device__ __forceinline__ uint32_t lane_bit(uint32_t low32, uint32_t seed) {
  return 1u << ((seed * low32) >> 27);
}

struct Block8 {
  uint32_t w[8];
};

__device__ __forceinline__ bool block_contains(const Block8& b, uint64_t hash) {
  const uint32_t low = static_cast<uint32_t>(hash);
  uint32_t missing = 0;
#pragma unroll
  for (int i = 0; i < kLanes; ++i) missing |= lane_bit(low, lane_seed(i)) & ~b.w[i];
  return missing == 0;
}

// ---- XXH64 key frontend (kHasherXxh64 = 1, hash.hpp:12; hash.cpp:45-114) ---
// The published XXH64 algorithm. hash_u64_key hashes the key's 8
// little-endian bytes (hash.cpp:108-114), which on device is the u64 itself.
constexpr uint64_t kXP1 = 0x9E3779B185EBCA87ull, kXP2 = 0xC2B2AE3D27D4EB4Full,
                   kXP3 = 0x165667B19E3779F9ull, kXP4 = 0x85EBCA77C2B2AE63ull,
                   kXP5 = 0x27D4EB2F165667C5ull;

__host__ __device__ __forceinline__ uint64_t xxh_rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__host__ __device__ __forceinline__ uint64_t xxh_round(uint64_t acc, uint64_t in) {
  return xxh_rotl(acc + in * kXP2, 31) * kXP1;
}
__host__ __device__ __forceinline__ uint64_t xxh_avalanche(uint64_t h) {
  h ^= h >> 33;
  h *= kXP2;
  h ^= h >> 29;
  h *= kXP3;
  return h ^ (h >> 32);
}

__host__ __device__ __forceinline__ uint64_t xxh64_u64(uint64_t key, uint64_t seed) {
  uint64_t h = seed + kXP5 + 8;
  h ^= xxh_round(0, key);
  h = xxh_rotl(h, 27) * kXP1 + kXP4;
  return xxh_avalanche(h);
}

__device__ __forceinline__ uint64_t xxh_load(const uint8_t* p, int bytes) {
  uint64_t v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// Arbitrary byte string (hash_key, hash.cpp:100-106).
__device__ inline uint64_t xxh64_bytes(const uint8_t* p, uint64_t len, uint64_t seed) {
  const uint8_t* end = p + len;
  uint64_t h;
  if (len >= 32) {
    uint64_t v1 = seed + kXP1 + kXP2, v2 = seed + kXP2, v3 = seed, v4 = seed - kXP1;
    do {
      v1 = xxh_round(v1, xxh_load(p, 8));
      v2 = xxh_round(v2, xxh_load(p + 8, 8));
      v3 = xxh_round(v3, xxh_load(p + 16, 8));
      v4 = xxh_round(v4, xxh_load(p + 24, 8));
      p += 32;
    } while (p + 32 <= end);
    h = xxh_rotl(v1, 1) + xxh_rotl(v2, 7) + xxh_rotl(v3, 12) + xxh_rotl(v4, 18);
    h = (h ^ xxh_round(0, v1)) * kXP1 + kXP4;
    h = (h ^ xxh_round(0, v2)) * kXP1 + kXP4;
    h = (h ^ xxh_round(0, v3)) * kXP1 + kXP4;
    h = (h ^ xxh_round(0, v4)) * kXP1 + kXP4;
  } else {
    h = seed + kXP5;
  }
  h += len;
  for (; p + 8 <= end; p += 8) h = xxh_rotl(h ^ xxh_round(0, xxh_load(p, 8)), 27) * kXP1 + kXP4;
  if (p + 4 <= end) {
    h = xxh_rotl(h ^ (xxh_load(p, 4) * kXP1), 23) * kXP2 + kXP3;
    p += 4;
  }
  for (; p < end; ++p) h = xxh_rotl(h ^ (*p * kXP5), 11) * kXP1;
  return xxh_avalanche(h);
}

// Key handling of the fused kernels: raw 64-bit hashes (kHasherRaw) or u64
// keys hashed on the fly with XXH64 (kHasherXxh64).
template <bool kKeys>
__device__ __forceinline__ uint64_t to_hash(uint64_t v, uint64_t seed) {
  if constexpr (kKeys) return xxh64_u64(v, seed);
  else return v;
}

// ---- memory primitives ---------------------------------------------------
// Streamed once (hash arrays): skip L1, evict-first in L2 so the stream does
// not push the filter out of L2.
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p, uint64_t policy) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
               : "=l"(v)
               : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t policy) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// One 32-byte block in a single 256-bit load (LDG.E.256), read-only path,
// no L1 allocation, evict-last in L2 (the filter is the reused working set).
__device__ __forceinline__ void ld_block_nc(const uint32_t* p, Block8& b) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_last.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
        "=r"(b.w[6]), "=r"(b.w[7])
      : "l"(p));
}

// Same without the L2 priority hint (blocked path: the working slice changes
// as the batch advances, so no line should outlive its slice).
__device__ __forceinline__ void ld_block_nc_normal(const uint32_t* p, Block8& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]),
                 "=r"(b.w[5]), "=r"(b.w[6]), "=r"(b.w[7])
               : "l"(p));
}

// Same, but L1-allocating (L2-resident filters get some L1 reuse).
__device__ __forceinline__ void ld_block_l1(const uint32_t* p, Block8& b) {
  asm volatile("ld.global.nc.L2::evict_last.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]),
                 "=r"(b.w[5]), "=r"(b.w[6]), "=r"(b.w[7])
               : "l"(p));
}

// Coherent-enough lane read for test-before-set inserts. A stale value can
// only claim a bit is clear when it is set (bits are monotone), which costs a
// redundant red, never a lost insert.
__device__ __forceinline__ uint32_t ld_lane(const uint32_t* p, uint64_t policy) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy));
  return v;
}

// Fire-and-forget atomic OR at L2 (REDG.E.OR.STRONG.GPU); `policy` is an L2
// cache policy from createpolicy (evict-last keeps the filter resident).
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v, uint64_t policy) {
  asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v),
               "l"(policy)
               : "memory");
}

__device__ __forceinline__ void red_or64(uint64_t* p, uint64_t v, uint64_t policy) {
  asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v),
               "l"(policy)
               : "memory");
}

__device__ __forceinline__ void red_or64_nohint(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_pair(const uint64_t* p, uint64_t policy) {
  uint64_t v;
  asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ void st_stream_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Output words that are not re-read soon (range-split bitmaps): evict-first
// in L2, so a pass's bitmap does not push the filter range it probes out of L2.
__device__ __forceinline__ void st_stream_u32_ef(uint32_t* p, uint32_t v, uint64_t policy) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(policy) : "memory");
}

__device__ __forceinline__ void st_stream_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.global.L1::no_allocate.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace dev
}  // namespace sbbf
