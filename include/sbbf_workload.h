/*
 * sbbf_workload.h — on-device generators for the seeded synthetic hash
 * streams of BASELINE.json's configs. Bench and test
 * plumbing, not part of the reference's API: they let bench.py materialise
 * billions of hashes directly in HBM. oracle/sbbf_oracle.c restates each
 * stream on the host, and tests/ check device == host prefixes.
 *
 * splitmix64(seed) output i = fmix(seed + (i+1) * 0x9e3779b97f4a7c15) — a
 * counter-based generator, so any index range is generated independently.
 */
#ifndef SBBF_WORKLOAD_H
#define SBBF_WORKLOAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is the only exported surface */
#endif

/* The insert stream of a config. Positions < fresh_prefix are fresh; a
 * position j >= fresh_prefix is a duplicate iff
 *   floor((j'+1) * dup_num / dup_den) > floor(j' * dup_num / dup_den),
 * j' = j - fresh_prefix. Fresh positions consume `seed` in order. A duplicate
 * takes the value of fresh position r, r = the first index with
 * u < zipf_cdf[r] (u = splitmix64(dup_sel_seed, j); r clamps to zipf_n-1).
 * dup_num == 0 means every position is fresh (configs 1, 2, 3, 5). */
typedef struct {
  uint64_t seed;
  uint64_t fresh_prefix;
  uint64_t dup_num, dup_den;
  uint64_t dup_sel_seed;
  const uint64_t* zipf_cdf; /* device pointer, zipf_n entries (dup streams only) */
  uint64_t zipf_n;
} sbbf_insert_stream_t;

/* out[k] = insert-stream value at position start + k. */
int sbbf_gen_inserts(const sbbf_insert_stream_t* s, uint64_t start, uint64_t n, uint64_t* d_out,
                     void* stream);

/* Mixed lookup stream: position j is a member iff
 * floor((j+1)p/q) > floor(jp/q); a member is the insert-stream value at
 * position mulhi64(splitmix64(sel_seed, j), num_inserts); non-members consume
 * nonmember_seed in order (index j - floor(jp/q)). */
int sbbf_gen_lookups(const sbbf_insert_stream_t* s, uint64_t num_inserts, uint64_t nonmember_seed,
                     uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start, uint64_t n,
                     uint64_t* d_out, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
