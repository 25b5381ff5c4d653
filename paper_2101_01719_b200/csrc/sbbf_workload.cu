// sbbf_workload.cu — device generators for BASELINE.json's synthetic hash
// streams (include/sbbf_workload.h). Bench/test plumbing: they let bench.py
// create inputs in HBM without a host round trip. The host restatement is
// oracle/sbbf_oracle.c (oracle_gen_*); tests check equal prefixes.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "sbbf_internal.h"

namespace sbbf {
namespace {

__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// floor(j * p / q) with a 128-bit intermediate (p, q < 2^63).
__device__ __forceinline__ uint64_t floor_frac(uint64_t j, uint64_t p, uint64_t q) {
  const uint64_t lo = j * p, hi = __umul64hi(j, p);
  if (hi == 0) return lo / q;
  // 128/64 division by long division on 64-bit halves (hi < q always here).
  uint64_t rem = hi, quot = 0;
  for (int b = 63; b >= 0; --b) {
    const bool carry = rem >> 63;
    rem = (rem << 1) | ((lo >> b) & 1u);
    if (carry || rem >= q) {
      rem -= q;
      quot |= uint64_t{1} << b;
    }
  }
  return quot;
}

struct Stream {
  uint64_t seed, fresh_prefix, dup_num, dup_den, dup_sel_seed;
  const uint64_t* zipf_cdf;
  uint64_t zipf_n;
};

__device__ uint64_t insert_value(const Stream& s, uint64_t j) {
  if (s.dup_num == 0 || j < s.fresh_prefix) return splitmix64_at(s.seed, j);
  const uint64_t jj = j - s.fresh_prefix;
  const uint64_t before = floor_frac(jj, s.dup_num, s.dup_den);
  if (floor_frac(jj + 1, s.dup_num, s.dup_den) == before) return splitmix64_at(s.seed, j - before);
  // Duplicate: inverse-CDF Zipf rank by binary search over integer thresholds.
  const uint64_t u = splitmix64_at(s.dup_sel_seed, j);
  uint64_t lo = 0, hi = s.zipf_n - 1;  // first r with u < cdf[r], clamped
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (u < s.zipf_cdf[mid])
      hi = mid;
    else
      lo = mid + 1;
  }
  return splitmix64_at(s.seed, lo);  // rank r < fresh_prefix is fresh position r
}

__global__ void gen_inserts_kernel(Stream s, uint64_t start, uint64_t n, uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride)
    out[k] = insert_value(s, start + k);
}

__global__ void gen_lookups_kernel(Stream s, uint64_t num_inserts, uint64_t nonmember_seed,
                                   uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start,
                                   uint64_t n, uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint64_t j = start + k;
    const uint64_t before = floor_frac(j, p, q);
    uint64_t v;
    if (floor_frac(j + 1, p, q) > before) {
      v = insert_value(s, __umul64hi(splitmix64_at(sel_seed, j), num_inserts));
    } else {
      v = splitmix64_at(nonmember_seed, j - before);
    }
    out[k] = v;
  }
}

Stream to_stream(const sbbf_insert_stream_t* s) {
  return Stream{s->seed, s->fresh_prefix, s->dup_num, s->dup_den, s->dup_sel_seed, s->zipf_cdf,
                s->zipf_n};
}

thread_local std::string g_gen_err;

int gen_rc(cudaError_t e) {
  if (e == cudaSuccess) return SBBF_OK;
  g_gen_err = cudaGetErrorString(e);
  return SBBF_ECUDA;
}

bool stream_ok(const sbbf_insert_stream_t* s) {
  if (!s) return false;
  if (s->dup_num != 0 && (s->dup_den == 0 || !s->zipf_cdf || s->zipf_n == 0 ||
                          s->zipf_n > s->fresh_prefix || s->dup_num > s->dup_den ||
                          s->dup_den >= (uint64_t{1} << 63)))
    return false;
  return true;
}

}  // namespace
}  // namespace sbbf

extern "C" {

int sbbf_gen_inserts(const sbbf_insert_stream_t* s, uint64_t start, uint64_t n, uint64_t* d_out,
                     void* stream) {
  if (!sbbf::stream_ok(s) || (n && !d_out)) return SBBF_EINVAL;
  if (n == 0) return SBBF_OK;
  sbbf::note_launch();
  const uint64_t g = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
  sbbf::gen_inserts_kernel<<<static_cast<unsigned>(g), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      sbbf::to_stream(s), start, n, d_out);
  return sbbf::gen_rc(cudaGetLastError());
}

int sbbf_gen_lookups(const sbbf_insert_stream_t* s, uint64_t num_inserts, uint64_t nonmember_seed,
                     uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start, uint64_t n,
                     uint64_t* d_out, void* stream) {
  if (!sbbf::stream_ok(s) || (n && !d_out) || q == 0 || p > q || q >= (uint64_t{1} << 63) ||
      (p > 0 && num_inserts == 0))
    return SBBF_EINVAL;
  if (n == 0) return SBBF_OK;
  sbbf::note_launch();
  const uint64_t g = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
  sbbf::gen_lookups_kernel<<<static_cast<unsigned>(g), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      sbbf::to_stream(s), num_inserts, nonmember_seed, sel_seed, p, q, start, n, d_out);
  return sbbf::gen_rc(cudaGetLastError());
}

}  // extern "C"
