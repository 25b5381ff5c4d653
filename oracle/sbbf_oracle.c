/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the SBBF hot path (see
 * sbbf_oracle.h for the contract: tests/, smoke() and bench.py's
 * cpu_baseline leg may use it, the product path never does).
 *
 * Every function cites the reference line it restates. Paths are relative to
 * /root/reference/proj/.
 */
#include "sbbf_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* core/include/sbbf/filter.hpp:18-21 — lane seeds, lane 0 first. */
static const uint32_t kSeeds[8] = {0x44974d91u, 0x47b6137bu, 0xa2b7289du, 0x8824ad5bu,
                                   0x2df1424bu, 0x705495c7u, 0x5c6bfb31u, 0x9efc4947u};

/* core/src/filter.cpp:15-29 (mul_high_u64) and :125-127 (block_index):
 * floor(hash * num_buckets / 2^64) over the full 128-bit product. */
uint64_t oracle_block_index(uint64_t hash, uint64_t num_buckets) {
  return (uint64_t)(((unsigned __int128)hash * (unsigned __int128)num_buckets) >> 64);
}

/* core/src/filter.cpp:129-138 (make_mask): lane i gets bit
 * (seed_i * low32(hash) mod 2^32) >> 27. */
void oracle_make_mask(uint64_t hash, uint32_t lanes[8]) {
  const uint32_t low = (uint32_t)hash;
  for (int i = 0; i < 8; ++i) lanes[i] = 1u << ((kSeeds[i] * low) >> 27);
}

/* core/src/filter.cpp:31-36 (add_scalar) via :184-194 (add_hashes). */
void oracle_add_hashes(uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                       uint64_t n) {
  for (uint64_t k = 0; k < n; ++k) {
    uint32_t m[8];
    oracle_make_mask(hashes[k], m);
    uint32_t* b = blocks + 8 * oracle_block_index(hashes[k], num_buckets);
    for (int i = 0; i < 8; ++i) b[i] |= m[i];
  }
}

/* core/src/filter.cpp:38-46 (find_scalar): all eight mask bits set, i.e.
 * (~block & mask) == 0; results are 0/1 bytes as in :196-207. */
static inline int find_one(const uint32_t* blocks, uint64_t num_buckets, uint64_t h) {
  uint32_t m[8];
  oracle_make_mask(h, m);
  const uint32_t* b = blocks + 8 * oracle_block_index(h, num_buckets);
  uint32_t missing = 0;
  for (int i = 0; i < 8; ++i) missing |= m[i] & ~b[i];
  return missing == 0;
}

void oracle_find_hashes(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                        uint64_t n, uint8_t* results) {
  for (uint64_t k = 0; k < n; ++k) results[k] = (uint8_t)find_one(blocks, num_buckets, hashes[k]);
}

/* tools/harness.cpp:173-200 — lookups sharded over contiguous key ranges
 * against one read-only filter. */
struct find_job {
  const uint32_t* blocks;
  uint64_t nb;
  const uint64_t* hashes;
  uint64_t begin, end;
  uint8_t* out;
};

static void* find_worker(void* arg) {
  struct find_job* j = (struct find_job*)arg;
  oracle_find_hashes(j->blocks, j->nb, j->hashes + j->begin, j->end - j->begin, j->out + j->begin);
  return NULL;
}

void oracle_find_hashes_mt(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                           uint64_t n, uint8_t* results, int threads) {
  if (threads <= 1) {
    oracle_find_hashes(blocks, num_buckets, hashes, n, results);
    return;
  }
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  struct find_job* jobs = (struct find_job*)calloc((size_t)threads, sizeof(struct find_job));
  for (int t = 0; t < threads; ++t) {
    jobs[t].blocks = blocks;
    jobs[t].nb = num_buckets;
    jobs[t].hashes = hashes;
    jobs[t].begin = n * (uint64_t)t / (uint64_t)threads;
    jobs[t].end = n * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].out = results;
    pthread_create(&tid[t], NULL, find_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
}

/* Packed form of the same answers: bit (k % 32) of word k / 32 is key k. */
void oracle_find_bits(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                      uint64_t n, uint32_t* bits) {
  memset(bits, 0, (size_t)((n + 31) / 32) * sizeof(uint32_t));
  for (uint64_t k = 0; k < n; ++k)
    if (find_one(blocks, num_buckets, hashes[k])) bits[k >> 5] |= 1u << (k & 31);
}

/* ---- FilterImage v1 --------------------------------------------------- */

/* core/src/persist.cpp:15-28 — reflected IEEE table, polynomial 0xEDB88320. */
static uint32_t crc_table[256];
static int crc_ready = 0;

static void crc_init(void) {
  if (crc_ready) return;
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
    crc_table[i] = c;
  }
  crc_ready = 1;
}

/* Raw register update (no pre/post inversion). */
uint32_t oracle_crc32_update(uint32_t state, const uint8_t* data, uint64_t len) {
  crc_init();
  for (uint64_t i = 0; i < len; ++i) state = (state >> 8) ^ crc_table[(state ^ data[i]) & 0xFFu];
  return state;
}

/* core/src/persist.cpp:64-70 (crc32_ieee). */
uint32_t oracle_crc32_ieee(const uint8_t* data, uint64_t len) {
  return oracle_crc32_update(0xFFFFFFFFu, data, len) ^ 0xFFFFFFFFu;
}

/* core/include/sbbf/persist.hpp:14-30 (layout, image_size). */
uint64_t oracle_image_size(uint64_t num_buckets) { return 17 + 32 * num_buckets + 4; }

static void put_le(uint8_t* p, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

static uint64_t get_le(const uint8_t* p, int bytes) {
  uint64_t v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

static void image_header(uint8_t hdr[17], uint64_t num_buckets, uint32_t hasher_id) {
  hdr[0] = 'S';
  hdr[1] = 'B';
  hdr[2] = 'B';
  hdr[3] = 'F';
  hdr[4] = 1; /* persist.hpp:21 kImageVersion */
  put_le(hdr + 5, hasher_id, 4);
  put_le(hdr + 9, num_buckets, 8);
}

/* core/src/persist.cpp:72-88 (serialize). Lanes are stored little-endian; on
 * a little-endian host the payload is the block array's own bytes. */
uint64_t oracle_serialize(const uint32_t* blocks, uint64_t num_buckets, uint32_t hasher_id,
                          uint8_t* out, uint64_t cap) {
  const uint64_t size = oracle_image_size(num_buckets);
  if (cap < size) return 0;
  image_header(out, num_buckets, hasher_id);
  for (uint64_t w = 0; w < 8 * num_buckets; ++w) put_le(out + 17 + 4 * w, blocks[w], 4);
  put_le(out + size - 4, oracle_crc32_ieee(out, size - 4), 4);
  return size;
}

/* Same CRC as the serialize() trailer without materialising the image. */
uint32_t oracle_image_crc(const uint32_t* blocks, uint64_t num_buckets, uint32_t hasher_id) {
  uint8_t hdr[17];
  image_header(hdr, num_buckets, hasher_id);
  uint32_t s = oracle_crc32_update(0xFFFFFFFFu, hdr, 17);
  s = oracle_crc32_update(s, (const uint8_t*)blocks, 32 * num_buckets);
  return s ^ 0xFFFFFFFFu;
}

/* core/src/persist.cpp:90-126 (deserialize), same check order and codes as
 * PersistErrc (persist.hpp:33-40). */
int oracle_deserialize(const uint8_t* bytes, uint64_t len, uint64_t* num_buckets,
                       uint32_t* hasher_id, uint32_t* blocks) {
  if (len < 21) return 1;
  if (memcmp(bytes, "SBBF", 4) != 0) return 2;
  if (bytes[4] != 1) return 3;
  const uint32_t hid = (uint32_t)get_le(bytes + 5, 4);
  const uint64_t nb = get_le(bytes + 9, 8);
  if (nb == 0) return 4;
  if (nb > (UINT64_MAX - 21) / 32 || len != oracle_image_size(nb)) return 1;
  if ((uint32_t)get_le(bytes + len - 4, 4) != oracle_crc32_ieee(bytes, len - 4)) return 5;
  *num_buckets = nb;
  *hasher_id = hid;
  if (blocks)
    for (uint64_t w = 0; w < 8 * nb; ++w) blocks[w] = (uint32_t)get_le(bytes + 17 + 4 * w, 4);
  return 0;
}

uint64_t oracle_popcount_blocks(const uint32_t* blocks, uint64_t num_buckets) {
  uint64_t c = 0;
  for (uint64_t w = 0; w < 8 * num_buckets; ++w) c += (uint64_t)__builtin_popcount(blocks[w]);
  return c;
}

/* ---- workload streams -------------------------------------------------- */

/* Counter-based splitmix64 (BASELINE.json configs): output
 * i of splitmix64(seed) is fmix(seed + (i+1) * golden-gamma). */
uint64_t oracle_splitmix64_at(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void oracle_gen_splitmix(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = oracle_splitmix64_at(seed, start + i);
}

static uint64_t floor_frac(uint64_t j, uint64_t p, uint64_t q) {
  return (uint64_t)(((unsigned __int128)j * p) / q);
}

/* Config 4's duplicate rule: positions >= fresh_prefix are duplicates by an
 * exact fraction; a duplicate's Zipf rank is the first r with u < cdf[r]. */
uint64_t oracle_insert_value(const oracle_stream_t* s, uint64_t j) {
  if (s->dup_num == 0 || j < s->fresh_prefix) return oracle_splitmix64_at(s->seed, j);
  const uint64_t jj = j - s->fresh_prefix;
  const uint64_t before = floor_frac(jj, s->dup_num, s->dup_den);
  if (floor_frac(jj + 1, s->dup_num, s->dup_den) == before)
    return oracle_splitmix64_at(s->seed, j - before);
  const uint64_t u = oracle_splitmix64_at(s->dup_sel_seed, j);
  /* upper_bound over [0, zipf_n - 1): count of thresholds <= u */
  uint64_t lo = 0, len = s->zipf_n - 1;
  while (len > 0) {
    const uint64_t half = len / 2;
    if (s->zipf_cdf[lo + half] <= u) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return oracle_splitmix64_at(s->seed, lo);
}

void oracle_gen_inserts(const oracle_stream_t* s, uint64_t start, uint64_t n, uint64_t* out) {
  for (uint64_t k = 0; k < n; ++k) out[k] = oracle_insert_value(s, start + k);
}

void oracle_gen_lookups(const oracle_stream_t* s, uint64_t num_inserts, uint64_t nonmember_seed,
                        uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start, uint64_t n,
                        uint64_t* out) {
  for (uint64_t k = 0; k < n; ++k) {
    const uint64_t j = start + k;
    const uint64_t before = floor_frac(j, p, q);
    if (floor_frac(j + 1, p, q) > before) {
      const uint64_t idx = oracle_block_index(oracle_splitmix64_at(sel_seed, j), num_inserts);
      out[k] = oracle_insert_value(s, idx);
    } else {
      out[k] = oracle_splitmix64_at(nonmember_seed, j - before);
    }
  }
}

void oracle_gen_mixed(uint64_t member_seed, uint64_t num_members, uint64_t nonmember_seed,
                      uint64_t sel_seed, uint64_t p, uint64_t q, uint64_t start, uint64_t n,
                      uint64_t* out) {
  const oracle_stream_t s = {member_seed, 0, 0, 1, 0, NULL, 0};
  oracle_gen_lookups(&s, num_members, nonmember_seed, sel_seed, p, q, start, n, out);
}

/* std::mt19937_64 — Matsumoto & Nishimura's MT19937-64 with the C++
 * standard's parameters, used by the reference tests (filter_test.cpp,
 * persist_test.cpp, acceptance.cpp) to draw hashes. */
void oracle_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out) {
  enum { NN = 312, MM = 156 };
  const uint64_t MATRIX_A = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull,
                 LM = 0x7FFFFFFFull;
  uint64_t mt[NN];
  int mti;
  mt[0] = seed;
  for (mti = 1; mti < NN; ++mti)
    mt[mti] = 6364136223846793005ull * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  for (uint64_t k = 0; k < n; ++k) {
    if (mti >= NN) {
      int i;
      uint64_t x;
      for (i = 0; i < NN - MM; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX_A : 0ull);
      }
      for (; i < NN - 1; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX_A : 0ull);
      }
      x = (mt[NN - 1] & UM) | (mt[0] & LM);
      mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX_A : 0ull);
      mti = 0;
    }
    uint64_t x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    out[k] = x;
  }
}

/* ---- XXH64 (core/src/hash.cpp:45-96; the published XXH64 algorithm) ---- */
static const uint64_t P1 = 11400714785074694791ull, P2 = 14029467366897019727ull,
                      P3 = 1609587929392839161ull, P4 = 9650029242287828579ull,
                      P5 = 2870177450012600261ull;

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static inline uint64_t xround(uint64_t acc, uint64_t in) {
  acc += in * P2;
  acc = rotl64(acc, 31);
  return acc * P1;
}
static inline uint64_t xmerge(uint64_t acc, uint64_t v) {
  acc ^= xround(0, v);
  return acc * P1 + P4;
}

uint64_t oracle_xxh64(const uint8_t* p, uint64_t len, uint64_t seed) {
  const uint8_t* end = p + len;
  uint64_t h;
  if (len >= 32) {
    uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
    const uint8_t* limit = end - 32;
    do {
      v1 = xround(v1, get_le(p, 8));
      v2 = xround(v2, get_le(p + 8, 8));
      v3 = xround(v3, get_le(p + 16, 8));
      v4 = xround(v4, get_le(p + 24, 8));
      p += 32;
    } while (p <= limit);
    h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
    h = xmerge(h, v1);
    h = xmerge(h, v2);
    h = xmerge(h, v3);
    h = xmerge(h, v4);
  } else {
    h = seed + P5;
  }
  h += len;
  while (p + 8 <= end) {
    h ^= xround(0, get_le(p, 8));
    h = rotl64(h, 27) * P1 + P4;
    p += 8;
  }
  if (p + 4 <= end) {
    h ^= get_le(p, 4) * P1;
    h = rotl64(h, 23) * P2 + P3;
    p += 4;
  }
  while (p < end) {
    h ^= (*p) * P5;
    h = rotl64(h, 11) * P1;
    ++p;
  }
  h ^= h >> 33;
  h *= P2;
  h ^= h >> 29;
  h *= P3;
  h ^= h >> 32;
  return h;
}
