/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the SBBF hot path.
 *
 * A plain-C restatement of the reference's split block Bloom filter
 * (arxiv 2101.01719; /root/reference/proj/core/src/filter.cpp) plus the
 * synthetic workload streams that BASELINE.json names. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker: the product path (paper_2101_01719_b200) never calls
 * into this library.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * the reference's own known-answer vectors (filter_test.cpp:22-33,66-99,
 * persist_test.cpp:42-47,81-111) and against golden fixtures produced by the
 * reference itself (oracle/_ref, built from /root/reference sources by
 * oracle/Makefile; fixtures in tests/golden/ with tests/golden/make_golden.py).
 */
#ifndef SBBF_ORACLE_H
#define SBBF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- hot-path semantics (filter.hpp / filter.cpp) ---------------------- */
uint64_t oracle_block_index(uint64_t hash, uint64_t num_buckets);
void oracle_make_mask(uint64_t hash, uint32_t lanes[8]);
void oracle_add_hashes(uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes, uint64_t n);
void oracle_find_hashes(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                        uint64_t n, uint8_t* results);
void oracle_find_hashes_mt(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                           uint64_t n, uint8_t* results, int threads);
void oracle_find_bits(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                      uint64_t n, uint32_t* bits);

/* ---- FilterImage v1 (persist.hpp / persist.cpp) ------------------------ */
uint32_t oracle_crc32_ieee(const uint8_t* data, uint64_t len);
uint32_t oracle_crc32_update(uint32_t state, const uint8_t* data, uint64_t len);
uint64_t oracle_image_size(uint64_t num_buckets);
uint64_t oracle_serialize(const uint32_t* blocks, uint64_t num_buckets, uint32_t hasher_id,
                          uint8_t* out, uint64_t cap);
uint32_t oracle_image_crc(const uint32_t* blocks, uint64_t num_buckets, uint32_t hasher_id);
/* 0 ok, else 1+PersistErrc: 1 truncated, 2 bad magic, 3 bad version,
 * 4 bad bucket count, 5 bad checksum. On success fills *num_buckets,
 * *hasher_id and (if blocks != NULL) copies the payload. */
int oracle_deserialize(const uint8_t* bytes, uint64_t len, uint64_t* num_buckets,
                       uint32_t* hasher_id, uint32_t* blocks);
uint64_t oracle_popcount_blocks(const uint32_t* blocks, uint64_t num_buckets);

/* ---- workload streams (BASELINE.json configs) -------- */
uint64_t oracle_splitmix64_at(uint64_t seed, uint64_t index);
void oracle_gen_splitmix(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out);
/* Mixed lookup stream: position j (absolute, from `start`) is a member iff
 * floor((j+1)p/q) > floor(jp/q); members are insert-stream values at index
 * mulhi64(splitmix(sel_seed, j), num_members); non-members consume
 * nonmember_seed in order. */
void oracle_gen_mixed(uint64_t member_seed, uint64_t num_members, uint64_t nonmember_seed,
                      uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start, uint64_t n,
                      uint64_t* out);
/* Insert stream with optional Zipf duplicates; the same definition as
 * include/sbbf_workload.h's sbbf_insert_stream_t (config 4). */
typedef struct {
  uint64_t seed;
  uint64_t fresh_prefix;
  uint64_t dup_num, dup_den;
  uint64_t dup_sel_seed;
  const uint64_t* zipf_cdf; /* host pointer */
  uint64_t zipf_n;
} oracle_stream_t;
uint64_t oracle_insert_value(const oracle_stream_t* s, uint64_t j);
void oracle_gen_inserts(const oracle_stream_t* s, uint64_t start, uint64_t n, uint64_t* out);
void oracle_gen_lookups(const oracle_stream_t* s, uint64_t num_inserts, uint64_t nonmember_seed,
                        uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start, uint64_t n,
                        uint64_t* out);
/* mt19937_64 (std::mt19937_64) outputs, to replay the reference tests' inputs. */
void oracle_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out);

/* ---- XXH64 key frontend (hash.cpp; "next" row 2) ---------------------- */
uint64_t oracle_xxh64(const uint8_t* data, uint64_t len, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
