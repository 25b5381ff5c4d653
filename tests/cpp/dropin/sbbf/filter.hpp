// Drop-in proof (test infrastructure): this header stands in for the
// reference's core/include/sbbf/filter.hpp when the reference's OWN callers
// — tests/acceptance/acceptance.cpp, tools/harness.cpp (run_bench,
// run_fpp_sim), core/src/model.cpp (sbbf_fpp_mc) and core/src/persist.cpp —
// are compiled unmodified from /root/reference and linked against the GPU
// library instead of core/src/filter.cpp (tests/cpp/Makefile). Every filter
// they build, probe, serialize and load then lives in HBM behind the C ABI
// (include/sbbf_gpu.h) via the header-only class in include/sbbf_gpu.hpp.
//
// The names below are the reference interface (filter.hpp:11-109); the
// behaviour behind them is the GPU's:
//   * Backend: the reference's only plug-in point (filter.hpp:49-53). kAuto /
//     kScalar / kVector all run the sm_100a kernels on device 0; the GPU
//     stands in for the "vector" backend, so vector_backend_available() is
//     true and no constructor throws the runtime_error of filter.cpp:107-118.
//   * blocks() returns a host copy (std::vector<Block>) instead of a span
//     over host memory: every reference caller consumes it inside one
//     full-expression or range-for (persist.cpp:81), which a temporary
//     vector satisfies.
//   * block_index / make_mask run the device kernels on one value.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "sbbf_gpu.hpp"

namespace sbbf {

inline constexpr std::size_t kLanesPerBlock = 8;
inline constexpr std::size_t kLaneBits = 32;
inline constexpr std::size_t kBlockBits = kLanesPerBlock * kLaneBits;
inline constexpr std::size_t kBlockBytes = kBlockBits / 8;

// The frozen lane seeds (filter.hpp:18-21), for callers that restate the
// mask (tests/unit/reference_filter.hpp); the GPU kernels carry their own copy.
inline constexpr std::array<std::uint32_t, kLanesPerBlock> kLaneSeeds = {
    0x44974d91u, 0x47b6137bu, 0xa2b7289du, 0x8824ad5bu, 0x2df1424bu, 0x705495c7u, 0x5c6bfb31u, 0x9efc4947u,
};

using Block = gpu::Block;

struct LaneMask {
  std::array<std::uint32_t, kLanesPerBlock> lanes{};
};

inline std::uint64_t block_index(std::uint64_t hash, std::uint64_t num_buckets) noexcept {
  std::uint64_t out = 0;
  if (sbbf_gpu_block_index_host(&hash, 1, num_buckets, &out, 0) != SBBF_OK) std::terminate();
  return out;
}

inline LaneMask make_mask(std::uint64_t hash) noexcept {
  LaneMask m;
  if (sbbf_gpu_make_mask_host(&hash, 1, m.lanes.data(), 0) != SBBF_OK) std::terminate();
  return m;
}

enum class Backend : std::uint8_t { kAuto, kScalar, kVector };

inline bool vector_backend_available() noexcept { return true; }

class SplitBlockFilter : public gpu::SplitBlockFilter {
 public:
  explicit SplitBlockFilter(std::uint64_t num_buckets, std::uint32_t hasher_id = 0,
                            Backend backend = Backend::kAuto)
      : gpu::SplitBlockFilter(num_buckets, hasher_id, /*device=*/0), backend_(backend) {}

  static SplitBlockFilter from_blocks(std::vector<Block> blocks, std::uint32_t hasher_id = 0,
                                      Backend backend = Backend::kAuto) {
    if (blocks.empty()) throw std::invalid_argument("SplitBlockFilter needs at least one bucket");
    SplitBlockFilter f(blocks.size(), hasher_id, backend);
    gpu::check(sbbf_gpu_from_host(f.handle(), blocks.data(), blocks.size() * sizeof(Block)), "from_blocks");
    return f;
  }

  Backend backend() const noexcept { return backend_ == Backend::kScalar ? Backend::kScalar : Backend::kVector; }

 private:
  Backend backend_;
};

}  // namespace sbbf
