// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// core (/root/reference/proj/core/src/{filter,persist,hash}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libsbbf_ref.so with the reference's
// Release flags (-std=c++20 -O3 -DNDEBUG, proj/CMakeLists.txt:7-9).
//
// Used (a) to pin the C restatement in sbbf_oracle.c and generate the golden
// fixtures under tests/golden/, and (b) as bench.py's CPU baseline
// (cpu_baseline.kind = "reference"): the timing loops below restate
// run_bench's method (tools/harness.cpp:132-245) — steady_clock around
// add_hashes on a fresh filter (1 thread, the only legal writer mode,
// filter.hpp:62-64) and around find_hashes sharded over std::jthread
// (harness.cpp:173-200).
#include <algorithm>
#include <chrono>
#include <random>
#include <cstdint>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "sbbf/filter.hpp"
#include "sbbf/hash.hpp"
#include "sbbf/model.hpp"
#include "sbbf/persist.hpp"

using sbbf::SplitBlockFilter;

namespace {
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }
}  // namespace

extern "C" {

uint64_t ref_block_index(uint64_t hash, uint64_t num_buckets) {
  return sbbf::block_index(hash, num_buckets);
}

void ref_make_mask(uint64_t hash, uint32_t* lanes) {
  const sbbf::LaneMask m = sbbf::make_mask(hash);
  for (int i = 0; i < 8; ++i) lanes[i] = m.lanes[i];
}

int ref_vector_backend_available(void) { return sbbf::vector_backend_available() ? 1 : 0; }

// backend: 0 auto, 1 scalar, 2 vector (filter.hpp:49-53). Returns NULL on
// the constructor's exceptions (num_buckets == 0, vector unavailable).
void* ref_filter_new(uint64_t num_buckets, uint32_t hasher_id, int backend) {
  try {
    return new SplitBlockFilter(num_buckets, hasher_id, static_cast<sbbf::Backend>(backend));
  } catch (...) {
    return nullptr;
  }
}

void ref_filter_free(void* f) { delete static_cast<SplitBlockFilter*>(f); }

void ref_filter_add(void* f, const uint64_t* hashes, uint64_t n) {
  static_cast<SplitBlockFilter*>(f)->add_hashes(std::span<const uint64_t>(hashes, n));
}

void ref_filter_add_one(void* f, uint64_t hash) { static_cast<SplitBlockFilter*>(f)->add_hash(hash); }

int ref_filter_find_one(void* f, uint64_t hash) {
  return static_cast<SplitBlockFilter*>(f)->find_hash(hash) ? 1 : 0;
}

void ref_filter_find(void* f, const uint64_t* hashes, uint64_t n, uint8_t* out) {
  static_cast<SplitBlockFilter*>(f)->find_hashes(std::span<const uint64_t>(hashes, n), out);
}

// harness.cpp:173-200: contiguous shards, one jthread each, shared filter.
void ref_filter_find_mt(void* f, const uint64_t* hashes, uint64_t n, uint8_t* out, int threads) {
  const SplitBlockFilter& filter = *static_cast<SplitBlockFilter*>(f);
  if (threads <= 1) {
    filter.find_hashes(std::span<const uint64_t>(hashes, n), out);
    return;
  }
  std::vector<std::jthread> workers;
  workers.reserve(threads);
  for (int t = 0; t < threads; ++t) {
    const uint64_t begin = n * t / threads, end = n * (t + 1) / threads;
    workers.emplace_back([&, begin, end] {
      filter.find_hashes(std::span<const uint64_t>(hashes + begin, end - begin), out + begin);
    });
  }
}

uint64_t ref_filter_num_buckets(void* f) { return static_cast<SplitBlockFilter*>(f)->num_buckets(); }

void ref_filter_blocks(void* f, uint32_t* out) {
  const auto blocks = static_cast<SplitBlockFilter*>(f)->blocks();
  std::memcpy(out, blocks.data(), blocks.size() * sizeof(sbbf::Block));
}

// from_blocks (filter.hpp:74-75)
void* ref_filter_from_blocks(const uint32_t* words, uint64_t num_buckets, uint32_t hasher_id) {
  try {
    std::vector<sbbf::Block> blocks(num_buckets);
    std::memcpy(blocks.data(), words, num_buckets * sizeof(sbbf::Block));
    return new SplitBlockFilter(SplitBlockFilter::from_blocks(std::move(blocks), hasher_id));
  } catch (...) {
    return nullptr;
  }
}

uint64_t ref_filter_serialize(void* f, uint8_t* out, uint64_t cap) {
  const std::vector<uint8_t> img = sbbf::serialize(*static_cast<SplitBlockFilter*>(f));
  if (cap < img.size()) return 0;
  std::memcpy(out, img.data(), img.size());
  return img.size();
}

// Returns 0 and a new filter in *out, or 1 + PersistErrc.
int ref_deserialize(const uint8_t* bytes, uint64_t len, void** out) {
  try {
    *out = new SplitBlockFilter(sbbf::deserialize(std::span<const uint8_t>(bytes, len)));
    return 0;
  } catch (const sbbf::PersistError& e) {
    return 1 + static_cast<int>(e.code());
  } catch (...) {
    return 99;
  }
}

uint32_t ref_crc32(const uint8_t* data, uint64_t len) {
  return sbbf::crc32_ieee(std::span<const uint8_t>(data, len));
}

uint64_t ref_hash_key(const uint8_t* data, uint64_t len, uint64_t seed) {
  return sbbf::hash_key(std::span<const uint8_t>(data, len), seed);
}

uint64_t ref_hash_u64_key(uint64_t key, uint64_t seed) { return sbbf::hash_u64_key(key, seed); }

// std::mt19937_64 draws, to replay the reference tests' hash inputs exactly.
void ref_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out) {
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng();
}

// run_fpp_sim's loop (tools/harness.cpp:84-97) with the reference's own
// hash_u64_key / add_hash / find_hash: counters [0, ndv) inserted, counters
// [2^32, 2^32 + queries) probed. Writes the false-positive count and the
// image CRC of the built filter (hasher id kHasherXxh64).
void ref_fpp_sim(uint64_t ndv, uint64_t num_buckets, uint64_t queries, uint64_t seed, uint64_t* fp,
                 uint32_t* image_crc) {
  SplitBlockFilter filter(num_buckets, sbbf::kHasherXxh64);
  for (uint64_t c = 0; c < ndv; ++c) filter.add_hash(sbbf::hash_u64_key(c, seed));
  uint64_t hits = 0;
  for (uint64_t i = 0; i < queries; ++i)
    hits += filter.find_hash(sbbf::hash_u64_key((uint64_t{1} << 32) + i, seed)) ? 1 : 0;
  *fp = hits;
  const std::vector<uint8_t> img = sbbf::serialize(filter);
  *image_crc = static_cast<uint32_t>(img[img.size() - 4]) | (static_cast<uint32_t>(img[img.size() - 3]) << 8) |
               (static_cast<uint32_t>(img[img.size() - 2]) << 16) | (static_cast<uint32_t>(img[img.size() - 1]) << 24);
}

// model.cpp:78-103,187-212 (sbbf_fpp, size_for) for the build tool's sizing.
double ref_sbbf_fpp(double a) { return sbbf::sbbf_fpp(a); }
double ref_standard_bloom_fpp(double bits_per_key, unsigned k) { return sbbf::standard_bloom_fpp(bits_per_key, k); }
unsigned ref_optimal_bloom_k(double bits_per_key) { return sbbf::optimal_bloom_k(bits_per_key); }

uint64_t ref_size_for(uint64_t ndv, double target_fpp) {
  try {
    return sbbf::size_for(ndv, target_fpp).num_buckets;
  } catch (...) {
    return 0;
  }
}

// ---- CPU baseline timing (harness.cpp:160-201) ---------------------------
// Each rep builds a fresh zeroed filter untimed, times add_hashes over the
// whole batch, then times find_hashes over the lookup batch with `threads`
// jthreads. Per-rep seconds are written to insert_s[rep] / lookup_s[rep];
// the last rep's filter stays alive in *keep (caller frees) for parity.
void ref_time_build_probe(uint64_t num_buckets, const uint64_t* inserts, uint64_t n_ins,
                          const uint64_t* lookups, uint64_t n_look, uint8_t* results, int threads,
                          int reps, double* insert_s, double* lookup_s, void** keep) {
  SplitBlockFilter* last = nullptr;
  for (int rep = 0; rep < reps; ++rep) {
    auto* fresh = new SplitBlockFilter(num_buckets);
    auto t0 = Clock::now();
    fresh->add_hashes(std::span<const uint64_t>(inserts, n_ins));
    insert_s[rep] = since(t0);
    t0 = Clock::now();
    ref_filter_find_mt(fresh, lookups, n_look, results, threads);
    lookup_s[rep] = since(t0);
    delete last;
    last = fresh;
  }
  if (keep) {
    *keep = last;
  } else {
    delete last;
  }
}

}  // extern "C"
