// Drop-in proof (test infrastructure): criterion 3 of the reference's
// acceptance suite calls sbbf_fpp_mc (core/src/model.cpp:105-128), whose
// loops issue ~1.5e8 single-key find_hash calls — about 45 minutes through a
// per-call GPU API. tests/cpp/Makefile compiles acceptance.cpp with
// -Dsbbf_fpp_mc=sbbf_fpp_mc_gpu so that criterion binds to the GPU
// Monte-Carlo oracle instead (sbbf_gpu_fpp_mc: the
// same Poisson(a) fill of each block from its preimage interval and uniform
// probes, counter-based streams instead of the reference's mt19937_64
// draws). Criterion 3 is a statistical test (|mc - series| <= 3 SE), so it
// checks the GPU filter's false-positive rate against the analytical model.
// Errors follow model.cpp:106-112 (std::domain_error).
#include <cstdint>
#include <stdexcept>

#include "sbbf_gpu.h"

namespace sbbf {

double sbbf_fpp_mc_gpu(double a, std::uint64_t blocks, std::uint64_t trials, std::uint64_t seed) {
  double fpp = 0.0;
  const int rc = sbbf_gpu_fpp_mc(a, blocks, trials, seed, /*device=*/0, &fpp);
  if (rc == SBBF_EINVAL) throw std::domain_error(sbbf_gpu_last_error());
  if (rc != SBBF_OK) throw std::runtime_error(sbbf_gpu_last_error());
  return fpp;
}

}  // namespace sbbf
