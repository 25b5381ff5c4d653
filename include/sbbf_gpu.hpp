// sbbf_gpu.hpp — header-only C++ drop-in over the C ABI (include/sbbf_gpu.h).
//
// Mirrors sbbf::SplitBlockFilter (/root/reference/proj/core/include/sbbf/
// filter.hpp:65-109): same member names, argument meaning and error
// behaviour, so reference callers (harness.cpp:163,169,189; model.cpp:119,125)
// switch by changing the type. Host spans go through the pipelined
// host-buffer path; raw device pointers have *_device overloads.
//
//   ctor(num_buckets, hasher_id)   throws std::invalid_argument on 0 buckets
//                                  (filter.cpp:160-162), std::runtime_error
//                                  when no CUDA device is usable
//   add_hash / find_hash           filter.hpp:77-78
//   add_hashes / find_hashes       filter.hpp:81-83 (results: 1 byte per key)
//   num_buckets / size_bytes       filter.hpp:85-86
//   blocks()                       filter.hpp:87 (returns a host copy)
//   hasher_id / set_hasher_id      filter.hpp:91-92
//   from_blocks                    filter.hpp:74-75
//   operator==                     filter.hpp:97-101
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sbbf_gpu.h"

namespace sbbf::gpu {

struct Block {
  std::array<std::uint32_t, 8> lanes{};
  friend bool operator==(const Block&, const Block&) = default;
};
static_assert(sizeof(Block) == 32);

[[noreturn]] inline void throw_status(int rc, const char* what) {
  const std::string msg = std::string(what) + ": " + sbbf_gpu_last_error();
  if (rc == SBBF_EINVAL) throw std::invalid_argument(msg);
  if (rc == SBBF_ENOMEM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

inline void check(int rc, const char* what) {
  if (rc != SBBF_OK) throw_status(rc, what);
}

class SplitBlockFilter {
 public:
  explicit SplitBlockFilter(std::uint64_t num_buckets, std::uint32_t hasher_id = 0, int device = 0) {
    check(sbbf_gpu_create(num_buckets, device, &h_), "SplitBlockFilter");
    if (hasher_id) check(sbbf_gpu_set_hasher_id(h_, hasher_id), "set_hasher_id");
  }

  static SplitBlockFilter from_blocks(const std::vector<Block>& blocks, std::uint32_t hasher_id = 0,
                                      int device = 0) {
    if (blocks.empty()) throw std::invalid_argument("SplitBlockFilter needs at least one bucket");
    SplitBlockFilter f(blocks.size(), hasher_id, device);
    check(sbbf_gpu_from_host(f.h_, blocks.data(), blocks.size() * sizeof(Block)), "from_blocks");
    return f;
  }

  SplitBlockFilter(SplitBlockFilter&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  SplitBlockFilter& operator=(SplitBlockFilter&& o) noexcept {
    if (this != &o) {
      sbbf_gpu_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  SplitBlockFilter(const SplitBlockFilter&) = delete;
  SplitBlockFilter& operator=(const SplitBlockFilter&) = delete;
  ~SplitBlockFilter() { sbbf_gpu_destroy(h_); }

  void add_hash(std::uint64_t hash) { check(sbbf_gpu_add_hash(h_, hash), "add_hash"); }
  bool find_hash(std::uint64_t hash) const {
    int found = 0;
    check(sbbf_gpu_find_hash(h_, hash, &found), "find_hash");
    return found != 0;
  }

  // Host spans (synchronous; copies pipelined with the kernels).
  void add_hashes(std::span<const std::uint64_t> hashes) {
    check(sbbf_gpu_add_hashes_host(h_, hashes.data(), hashes.size()), "add_hashes");
  }
  void find_hashes(std::span<const std::uint64_t> hashes, std::uint8_t* results) const {
    check(sbbf_gpu_find_hashes_host(h_, hashes.data(), hashes.size(), results), "find_hashes");
  }
  std::vector<std::uint8_t> find_hashes(std::span<const std::uint64_t> hashes) const {
    std::vector<std::uint8_t> out(hashes.size());
    find_hashes(hashes, out.data());
    return out;
  }

  // Device pointers (asynchronous on `stream`).
  void add_hashes_device(const std::uint64_t* d_hashes, std::uint64_t n, void* stream = nullptr) {
    check(sbbf_gpu_insert_batch(h_, d_hashes, n, stream), "insert_batch");
  }
  void find_hashes_device(const std::uint64_t* d_hashes, std::uint64_t n, std::uint8_t* d_results,
                          void* stream = nullptr) const {
    check(sbbf_gpu_find_batch(h_, d_hashes, n, d_results, stream), "find_batch");
  }
  void find_bits_device(const std::uint64_t* d_hashes, std::uint64_t n, std::uint32_t* d_bits,
                        void* stream = nullptr) const {
    check(sbbf_gpu_find_batch_bits(h_, d_hashes, n, d_bits, stream), "find_batch_bits");
  }

  std::uint64_t num_buckets() const noexcept { return sbbf_gpu_num_buckets(h_); }
  std::uint64_t size_bytes() const noexcept { return sbbf_gpu_size_bytes(h_); }
  std::vector<Block> blocks() const {
    std::vector<Block> out(num_buckets());
    check(sbbf_gpu_to_host(h_, out.data(), out.size() * sizeof(Block)), "blocks");
    return out;
  }
  std::uint32_t hasher_id() const noexcept { return sbbf_gpu_hasher_id(h_); }
  void set_hasher_id(std::uint32_t id) { check(sbbf_gpu_set_hasher_id(h_, id), "set_hasher_id"); }
  sbbf_gpu_t* handle() const noexcept { return h_; }

  friend bool operator==(const SplitBlockFilter& a, const SplitBlockFilter& b) {
    return a.hasher_id() == b.hasher_id() && a.blocks() == b.blocks();
  }

  // XXH64 frontend (kHasherXxh64, hash.hpp:12): u64 keys hashed in-kernel.
  void add_keys_device(const std::uint64_t* d_keys, std::uint64_t n, std::uint64_t seed = 0,
                       void* stream = nullptr) {
    check(sbbf_gpu_insert_keys_u64(h_, d_keys, n, seed, stream), "insert_keys_u64");
  }
  void find_keys_device(const std::uint64_t* d_keys, std::uint64_t n, std::uint8_t* d_results,
                        std::uint64_t seed = 0, void* stream = nullptr) const {
    check(sbbf_gpu_find_keys_u64(h_, d_keys, n, seed, d_results, stream), "find_keys_u64");
  }

  static SplitBlockFilter adopt(sbbf_gpu_t* h) {
    SplitBlockFilter f;
    f.h_ = h;
    return f;
  }

 private:
  SplitBlockFilter() = default;
  sbbf_gpu_t* h_ = nullptr;
};

// --- multi-GPU: one rank's view of a block-range sharded filter -------------
// (sbbf_dist_*; the reference has no distributed mode). Collective calls:
// every rank of the NCCL communicator calls them in the same order.
class ShardedFilter {
 public:
  ShardedFilter(void* nccl_comm, std::uint64_t total_buckets, std::uint64_t max_batch, int device = 0) {
    if (total_buckets == 0) throw std::invalid_argument("SplitBlockFilter needs at least one bucket");
    check(sbbf_dist_create(nccl_comm, total_buckets, max_batch, device, &d_), "ShardedFilter");
    total_ = total_buckets;
  }
  ShardedFilter(const ShardedFilter&) = delete;
  ShardedFilter& operator=(const ShardedFilter&) = delete;
  ~ShardedFilter() { sbbf_dist_destroy(d_); }

  int rank() const noexcept { return sbbf_dist_rank(d_); }
  int world() const noexcept { return sbbf_dist_world(d_); }
  void add_hashes_device(const std::uint64_t* d_hashes, std::uint64_t n, void* stream = nullptr) {
    check(sbbf_dist_insert(d_, d_hashes, n, stream), "sbbf_dist_insert");
  }
  void find_hashes_device(const std::uint64_t* d_hashes, std::uint64_t n, std::uint8_t* d_results,
                          void* stream = nullptr) {
    check(sbbf_dist_find(d_, d_hashes, n, d_results, stream), "sbbf_dist_find");
  }
  void find_bits_device(const std::uint64_t* d_hashes, std::uint64_t n, std::uint32_t* d_bits,
                        void* stream = nullptr) {
    check(sbbf_dist_find_bits(d_, d_hashes, n, d_bits, stream), "sbbf_dist_find_bits");
  }
  // The whole filter (the shards in rank order) on `root`; empty elsewhere.
  std::vector<Block> blocks(int root = 0) {
    std::vector<Block> out(rank() == root ? total_ : 0);
    check(sbbf_dist_gather(d_, out.data(), root), "sbbf_dist_gather");
    return out;
  }

 private:
  sbbf_dist_t* d_ = nullptr;
  std::uint64_t total_ = 0;
};

// --- persist.hpp:33-66 mirror (FilterImage v1; CRC computed on the GPU) ----
enum class PersistErrc { kTruncated, kBadMagic, kBadVersion, kBadBucketCount, kBadChecksum, kIo };

class PersistError : public std::runtime_error {
 public:
  PersistError(PersistErrc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  PersistErrc code() const noexcept { return code_; }

 private:
  PersistErrc code_;
};

[[noreturn]] inline void throw_persist(int rc, int errc, const char* what) {
  if (rc == SBBF_EFORMAT && errc >= 1 && errc <= 6)
    throw PersistError(static_cast<PersistErrc>(errc - 1), std::string(what) + ": " + sbbf_gpu_last_error());
  throw_status(rc, what);
}

inline std::vector<std::uint8_t> serialize(const SplitBlockFilter& f) {
  std::vector<std::uint8_t> out(sbbf_gpu_image_size(f.num_buckets()));
  std::uint64_t written = 0;
  check(sbbf_gpu_serialize(f.handle(), out.data(), out.size(), &written), "serialize");
  return out;
}

inline SplitBlockFilter deserialize(std::span<const std::uint8_t> bytes, int device = 0) {
  sbbf_gpu_t* h = nullptr;
  int errc = 0;
  const int rc = sbbf_gpu_deserialize(bytes.data(), bytes.size(), device, &h, &errc);
  if (rc != SBBF_OK) throw_persist(rc, errc, "deserialize");
  return SplitBlockFilter::adopt(h);
}

inline void save_filter(const SplitBlockFilter& f, const std::string& path) {
  int errc = 0;
  const int rc = sbbf_gpu_save(f.handle(), path.c_str(), &errc);
  if (rc != SBBF_OK) throw_persist(rc, errc, "save_filter");
}

inline SplitBlockFilter load_filter(const std::string& path, int device = 0) {
  sbbf_gpu_t* h = nullptr;
  int errc = 0;
  const int rc = sbbf_gpu_load(path.c_str(), device, &h, &errc);
  if (rc != SBBF_OK) throw_persist(rc, errc, "load_filter");
  return SplitBlockFilter::adopt(h);
}

}  // namespace sbbf::gpu
