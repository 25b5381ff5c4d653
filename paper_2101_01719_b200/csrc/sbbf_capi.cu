// sbbf_capi.cu — the C ABI declared in include/sbbf_gpu.h.
//
// Replaces sbbf::SplitBlockFilter (/root/reference/proj/core/include/sbbf/
// filter.hpp:65-109) for batched build and probe. The handle owns one
// cudaMalloc'd block array (256-byte aligned, so every 32-byte block is
// 32-byte aligned as the reference's alignas(32) Block requires,
// filter.hpp:25). No exceptions cross this boundary; every failure becomes a
// negative SBBF_E* code plus a thread-local message.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "sbbf_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace sbbf {
// Other translation units (sbbf_route.cu) report through sbbf_gpu_last_error.
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace sbbf

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  const int code = (e == cudaErrorMemoryAllocation) ? SBBF_ENOMEM
                   : (e == cudaErrorNoDevice || e == cudaErrorInvalidDevice ||
                      e == cudaErrorInsufficientDriver)
                       ? SBBF_ENODEV
                       : SBBF_ECUDA;
  return fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

// Makes `dev` current for the scope of an ABI call and restores the caller's.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

constexpr uint64_t kHostChunk = uint64_t{1} << 22;  // keys per pipelined host chunk (32 MiB): per-copy overheads outweigh a longer tail (e2e 2^18: 5.69, 2^20: 6.38, 2^22: 6.44 Gkeys/s)
constexpr int kHostStreams = 3;                      // chunks in flight: H2D / kernel / D2H

}  // namespace

struct sbbf_gpu {
  sbbf::DeviceInfo di;
  uint64_t nb = 0;                    // local block count (== geom.nb_local)
  sbbf::Geom geom{0, 0, 0};           // global bucket count / first block of this shard
  uint32_t* d_blocks = nullptr;
  uint32_t hasher_id = 0;
  int insert_variant = SBBF_INSERT_AUTO;
  int find_variant = SBBF_FIND_AUTO;
  // Host-buffer path resources, created on first use.
  std::mutex host_mu;
  bool host_ready = false;
  cudaStream_t hs[kHostStreams] = {};
  uint64_t* d_stage[kHostStreams] = {};
  void* d_res[kHostStreams] = {};
  uint64_t* h_one = nullptr;  // single-key slot [hash, result]: pinned host memory, mapped
  uint64_t* d_one = nullptr;  // ... and its device alias
  // L2-blocked path: filter slice bounds (global block ids), created lazily.
  std::mutex plan_mu;
  sbbf::BlockedPlan plan;
  uint64_t* d_plan_bounds = nullptr;
  uint64_t* d_super_bounds = nullptr;
};

namespace {

// Blocked path slice size: the slice being probed stays L2-resident while its
// keys stream by. On config 4 (1 GiB): 32 MiB slices 84.4 / 48.3 Gkeys/s
// (lookup / insert), 16 MiB 81.6 / 47.8, 64 MiB 68.7 / 38.0, 8 MiB 46.4 / 35.0
// (scripts/variant_ab.py; bucket counts round up to powers of two).
constexpr uint64_t kSliceBytes = 32ull << 20;
// SBBF_SLICE_MB overrides the slice size (A/B measurements only).
uint64_t slice_bytes() {
  static const uint64_t v = [] {
    const char* e = getenv("SBBF_SLICE_MB");
    const long mb = e ? atol(e) : 0;
    return mb > 0 ? static_cast<uint64_t>(mb) << 20 : kSliceBytes;
  }();
  return v;
}

// Blocked inserts pay once random atomics mostly miss L2: into a ~L2-sized
// filter (config 3) plain reds hit L2 often enough that the partition passes
// cost more than they save (39.1 vs 55.8 Gkeys/s). Lookups switch earlier
// (resolve_find). Both need at least half a key per block, or the slices'
// lines are fetched for too few keys.
bool blocked_pays(const sbbf_gpu* f, uint64_t n) {
  return f->nb * 32 > 2 * static_cast<uint64_t>(f->di.l2_bytes) && n >= f->nb / 2;
}

int resolve_insert(const sbbf_gpu* f, uint64_t n) {
  if (f->insert_variant != SBBF_INSERT_AUTO) return f->insert_variant;
  // Up to ~2x L2 (config 3's 128 MiB: much of it stays L2-resident) the
  // inserts are bound by the L2 atomic unit (op count): plain 64-bit reds
  // (51.5 vs 45.4 G/s with test-before-set, scripts/variant_ab.py). Beyond,
  // a batch of at least half a key per block is grouped by filter slice
  // first (blocked path, sbbf_blocked.cu); smaller batches load the lane pair
  // first (a load fills L2 faster than a missing atomic, and duplicates /
  // hot keys skip the atomic entirely: 22 vs 8 G/s on config 4).
  if (f->nb * 32 <= 2 * static_cast<uint64_t>(f->di.l2_bytes)) return SBBF_INSERT_WIDE;
  return blocked_pays(f, n) ? SBBF_INSERT_BLOCKED : SBBF_INSERT_WIDE_TEST;
}

bool smem_fits(const sbbf_gpu* f) {
  const uint64_t bytes = f->nb * 32;
  return bytes + 1024 <= f->di.smem_optin && bytes <= (200u << 10);
}

int resolve_find(const sbbf_gpu* f, uint64_t n) {
  if (f->find_variant == SBBF_FIND_SMEM && smem_fits(f)) return SBBF_FIND_SMEM;
  if (f->find_variant == SBBF_FIND_BLOCKED) return SBBF_FIND_BLOCKED;
  if (f->find_variant != SBBF_FIND_AUTO) return SBBF_FIND_GLOBAL;
  // Staging the filter costs one filter-size copy per CTA; it pays once each
  // SM probes enough keys to amortise it.
  if (smem_fits(f) && n >= 64 * f->nb) return SBBF_FIND_SMEM;
  // A whole filter up to ~1.2 x L2 is probed directly in two range-split
  // passes (config 3: 137.6 vs 112.8 Gkeys/s blocked, sbbf_kernels.cu
  // split_log2). Beyond, lookups gain from blocking as soon as the batch
  // has half a key per block; inserts only beyond 2 x L2 (resolve_insert).
  if (sbbf::split_log2(f->di, f->geom, true) > 0) return SBBF_FIND_GLOBAL;
  if (f->nb * 32 > static_cast<uint64_t>(f->di.l2_bytes) && n >= f->nb / 2) return SBBF_FIND_BLOCKED;
  return SBBF_FIND_GLOBAL;
}

// Slice bounds for the blocked path: parts slices of ~kSliceBytes over this
// shard's blocks, as global block ids (the partition kernel compares
// block_index against them).
int ensure_plan(sbbf_gpu* f) {
  std::lock_guard<std::mutex> lock(f->plan_mu);
  if (f->d_plan_bounds) return SBBF_OK;
  uint64_t parts = (f->nb * 32 + slice_bytes() - 1) / slice_bytes();
  // beyond 128 slices (chunk-local bucket ids are <= 7 bits, filters beyond
  // 4 GiB): super-slices of <= 128 slices (the super partition takes <= 64)
  uint64_t super = (parts + 127) / 128;
  super = super > 64 ? 64 : super;
  if (super > 1) parts = (parts + super - 1) / super;
  parts = parts < 2 ? 2 : (parts > 128 ? 128 : parts);
  uint64_t pow2 = 1;
  while (pow2 < parts) pow2 <<= 1;  // a power of two lets the partition use the hash's top bits
  parts = pow2;
  if (parts > f->nb) parts = f->nb;
  if (super > 1) {
    std::vector<uint64_t> sb(super + 1);
    for (uint64_t k = 0; k <= super; ++k)
      sb[k] = static_cast<uint64_t>((static_cast<unsigned __int128>(f->nb) * k) / super);
    cudaError_t e = cudaMalloc(&f->d_super_bounds, super * sizeof(uint64_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(f->d_super_bounds, sb.data(), super * sizeof(uint64_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(f->d_super_bounds);
      f->d_super_bounds = nullptr;
      return cuda_fail(e, "blocked plan");
    }
    f->plan.super_parts = static_cast<uint32_t>(super);
    f->plan.d_super_bounds = f->d_super_bounds;
    f->plan.h_super_bounds = sb;
  }
  std::vector<uint64_t> b(parts);
  for (uint64_t k = 0; k < parts; ++k)
    b[k] = f->geom.first + static_cast<uint64_t>((static_cast<unsigned __int128>(f->nb) * k) / parts);
  cudaError_t e = cudaMalloc(&f->d_plan_bounds, parts * sizeof(uint64_t));
  if (e == cudaSuccess)
    e = cudaMemcpy(f->d_plan_bounds, b.data(), parts * sizeof(uint64_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(f->d_plan_bounds);
    f->d_plan_bounds = nullptr;
    return cuda_fail(e, "blocked plan");
  }
  // Keep freed scratch in the stream-ordered pool between calls.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, f->di.device) == cudaSuccess) {
    uint64_t keep = ~uint64_t{0};
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  f->plan.parts = static_cast<uint32_t>(parts);
  f->plan.d_bounds = f->d_plan_bounds;
  f->plan.ctx = sbbf::blocked_ctx_create();  // scratch arena + side stream (null: pool scratch)
  return SBBF_OK;
}

// One dispatch point for every insert / find launch of the ABI.
cudaError_t do_insert(sbbf_gpu* f, int variant, const uint64_t* h, uint64_t n, cudaStream_t s) {
  if (variant == SBBF_INSERT_BLOCKED) {
    if (ensure_plan(f) != SBBF_OK) return cudaErrorMemoryAllocation;
    return sbbf::blocked_insert(f->di, f->d_blocks, f->geom, f->plan, h, n, s);
  }
  return sbbf::launch_insert(f->di, variant, f->d_blocks, f->geom, h, n, s);
}

cudaError_t do_find(sbbf_gpu* f, int variant, const uint64_t* h, uint64_t n, void* out, bool bits,
                    cudaStream_t s) {
  if (variant == SBBF_FIND_BLOCKED) {
    if (ensure_plan(f) != SBBF_OK) return cudaErrorMemoryAllocation;
    return sbbf::blocked_find(f->di, f->d_blocks, f->geom, f->plan, h, n, out, bits, s,
                              f->find_variant == SBBF_FIND_AUTO);
  }
  return sbbf::launch_find(f->di, variant, f->d_blocks, f->geom, h, n, out, bits, s);
}

int ensure_host_path(sbbf_gpu* f) {
  if (f->host_ready) return SBBF_OK;
  for (int i = 0; i < kHostStreams; ++i) {
    cudaError_t e = cudaStreamCreateWithFlags(&f->hs[i], cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    e = cudaMalloc(&f->d_stage[i], kHostChunk * sizeof(uint64_t));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
    e = cudaMalloc(&f->d_res[i], kHostChunk);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(results)");
  }
  f->host_ready = true;
  return SBBF_OK;
}

// The host-buffer pipeline: chunk c goes H2D -> kernel -> (D2H) on stream
// c % kHostStreams, so chunk c+1's upload overlaps chunk c's kernel and
// download (the copy engines are full duplex).
enum class HostOp { kInsert, kFindBytes, kFindBits };

int host_pipeline(sbbf_gpu* f, HostOp op, const uint64_t* h_hashes, uint64_t n, void* h_out) {
  if (n == 0) return SBBF_OK;
  if (!h_hashes || (op != HostOp::kInsert && !h_out)) return fail(SBBF_EINVAL, "null host buffer");
  std::lock_guard<std::mutex> lock(f->host_mu);
  DeviceGuard g(f->di.device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  int rc = ensure_host_path(f);
  if (rc != SBBF_OK) return rc;
  // The host calls are synchronous, like to_host: they start behind every
  // piece of work already queued on the device (the library's own streams
  // are non-blocking, so an insert the caller queued on its stream would not
  // otherwise be ordered before these lookups).
  cudaError_t e0 = cudaDeviceSynchronize();
  if (e0 != cudaSuccess) return cuda_fail(e0, "cudaDeviceSynchronize");
  for (uint64_t off = 0, c = 0; off < n; off += kHostChunk, ++c) {
    const uint64_t m = (n - off < kHostChunk) ? n - off : kHostChunk;
    const int s = static_cast<int>(c % kHostStreams);
    cudaError_t e = cudaMemcpyAsync(f->d_stage[s], h_hashes + off, m * sizeof(uint64_t),
                                    cudaMemcpyHostToDevice, f->hs[s]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    if (op == HostOp::kInsert) {
      e = do_insert(f, resolve_insert(f, m), f->d_stage[s], m, f->hs[s]);
      if (e != cudaSuccess) return cuda_fail(e, "insert kernel");
    } else {
      const bool bits = op == HostOp::kFindBits;
      e = do_find(f, resolve_find(f, m), f->d_stage[s], m, f->d_res[s], bits, f->hs[s]);
      if (e != cudaSuccess) return cuda_fail(e, "find kernel");
      // kHostChunk is a multiple of 32, so chunk bitmaps tile the output.
      void* dst = bits ? static_cast<void*>(static_cast<uint32_t*>(h_out) + off / 32)
                       : static_cast<void*>(static_cast<uint8_t*>(h_out) + off);
      const size_t bytes = bits ? ((m + 31) / 32) * sizeof(uint32_t) : m;
      e = cudaMemcpyAsync(dst, f->d_res[s], bytes, cudaMemcpyDeviceToHost, f->hs[s]);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    }
  }
  for (int s = 0; s < kHostStreams; ++s) {
    cudaError_t e = cudaStreamSynchronize(f->hs[s]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  }
  return SBBF_OK;
}

}  // namespace

namespace sbbf {

int gpu_insert_regions(sbbf_gpu_t* f, const uint64_t* const* keys, const uint64_t* counts, uint32_t nr,
                       cudaStream_t s, bool* handled) {
  *handled = false;
  uint64_t total = 0;
  for (uint32_t r = 0; r < nr; ++r) total += counts[r];
  if (total == 0) {
    *handled = true;
    return SBBF_OK;
  }
  if (resolve_insert(f, total) != SBBF_INSERT_BLOCKED) return SBBF_OK;
  DeviceGuard g(f->di.device);
  if (ensure_plan(f) != SBBF_OK) return SBBF_ENOMEM;
  const cudaError_t e = blocked_insert_regions(f->di, f->d_blocks, f->geom, f->plan, keys, counts, nr, s);
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return SBBF_OK;
  }
  *handled = true;
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "blocked_insert_regions");
}

int gpu_find_regions(const sbbf_gpu_t* fc, const uint64_t* const* keys, const uint64_t* counts, uint32_t nr,
                     uint8_t* const* outs, cudaStream_t s, bool* handled) {
  auto* f = const_cast<sbbf_gpu*>(fc);
  *handled = false;
  uint64_t total = 0;
  for (uint32_t r = 0; r < nr; ++r) total += counts[r];
  if (total == 0) {
    *handled = true;
    return SBBF_OK;
  }
  if (resolve_find(f, total) != SBBF_FIND_BLOCKED) return SBBF_OK;
  DeviceGuard g(f->di.device);
  if (ensure_plan(f) != SBBF_OK) return SBBF_ENOMEM;
  const cudaError_t e = blocked_find_regions(f->di, f->d_blocks, f->geom, f->plan, keys, counts, nr, outs, s,
                                             f->find_variant == SBBF_FIND_AUTO);
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return SBBF_OK;
  }
  *handled = true;
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "blocked_find_regions");
}

}  // namespace sbbf


extern "C" {

int sbbf_gpu_abi_version(void) { return SBBF_GPU_ABI_VERSION; }
const char* sbbf_gpu_last_error(void) { return g_err.c_str(); }
uint64_t sbbf_gpu_launch_count(void) { return sbbf::launch_count(); }

int sbbf_gpu_create(uint64_t num_buckets, int device, sbbf_gpu_t** out) {
  return sbbf_gpu_create_shard(num_buckets, 0, num_buckets, device, out);
}

int sbbf_gpu_create_shard(uint64_t total_buckets, uint64_t first_block, uint64_t num_buckets,
                          int device, sbbf_gpu_t** out) {
  if (!out) return fail(SBBF_EINVAL, "out is null");
  *out = nullptr;
  if (num_buckets == 0) return fail(SBBF_EINVAL, "SplitBlockFilter needs at least one bucket");
  if (num_buckets > (~uint64_t{0}) / 32) return fail(SBBF_EINVAL, "num_buckets overflows size");
  if (first_block > total_buckets || num_buckets > total_buckets - first_block)
    return fail(SBBF_EINVAL, "shard range exceeds total_buckets");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    return fail(SBBF_ENODEV, std::string("no CUDA device: ") +
                                 (e == cudaSuccess ? "count is 0" : cudaGetErrorString(e)));
  }
  if (device < 0 || device >= count) return fail(SBBF_ENODEV, "bad device ordinal");
  DeviceGuard g(device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  sbbf_gpu* f = new (std::nothrow) sbbf_gpu;
  if (!f) return fail(SBBF_ENOMEM, "host allocation failed");
  f->nb = num_buckets;
  f->geom = sbbf::Geom{total_buckets, first_block, num_buckets};
  f->di.device = device;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) == cudaSuccess) f->di.sms = v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) == cudaSuccess)
    f->di.smem_optin = static_cast<size_t>(v);
  if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device) == cudaSuccess)
    f->di.l2_bytes = static_cast<size_t>(v);
  e = cudaMalloc(&f->d_blocks, num_buckets * 32);
  if (e == cudaSuccess) e = cudaMemset(f->d_blocks, 0, num_buckets * 32);
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&f->h_one), 2 * sizeof(uint64_t), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&f->d_one), f->h_one, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    const int rc = cuda_fail(e, "allocating the block array");
    sbbf_gpu_destroy(f);
    return rc;
  }
  *out = f;
  return SBBF_OK;
}

int sbbf_gpu_destroy(sbbf_gpu_t* f) {
  if (!f) return SBBF_OK;
  {
    DeviceGuard g(f->di.device);
    if (f->d_blocks) cudaDeviceSynchronize();
    cudaFree(f->d_blocks);
    if (f->h_one) cudaFreeHost(f->h_one);
    sbbf::blocked_ctx_destroy(f->plan.ctx);
    cudaFree(f->d_plan_bounds);
    cudaFree(f->d_super_bounds);
    for (int i = 0; i < kHostStreams; ++i) {
      if (f->hs[i]) cudaStreamDestroy(f->hs[i]);
      cudaFree(f->d_stage[i]);
      cudaFree(f->d_res[i]);
    }
  }
  delete f;
  return SBBF_OK;
}

int sbbf_gpu_clear(sbbf_gpu_t* f, void* stream) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  DeviceGuard g(f->di.device);
  cudaError_t e = cudaMemsetAsync(f->d_blocks, 0, f->nb * 32, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "cudaMemsetAsync");
}

uint64_t sbbf_gpu_num_buckets(const sbbf_gpu_t* f) { return f ? f->nb : 0; }
uint64_t sbbf_gpu_total_buckets(const sbbf_gpu_t* f) { return f ? f->geom.nb_global : 0; }
uint64_t sbbf_gpu_first_block(const sbbf_gpu_t* f) { return f ? f->geom.first : 0; }
uint64_t sbbf_gpu_size_bytes(const sbbf_gpu_t* f) { return f ? f->nb * 32 : 0; }
uint32_t sbbf_gpu_hasher_id(const sbbf_gpu_t* f) { return f ? f->hasher_id : 0; }
int sbbf_gpu_device(const sbbf_gpu_t* f) { return f ? f->di.device : -1; }
void* sbbf_gpu_device_blocks(sbbf_gpu_t* f) { return f ? f->d_blocks : nullptr; }

int sbbf_gpu_set_hasher_id(sbbf_gpu_t* f, uint32_t hasher_id) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  f->hasher_id = hasher_id;
  return SBBF_OK;
}

int sbbf_gpu_insert_batch(sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n, void* stream) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  if (n == 0) return SBBF_OK;  // empty batch is a no-op (filter_test.cpp:169-175)
  if (!d_hashes) return fail(SBBF_EINVAL, "null hashes");
  DeviceGuard g(f->di.device);
  cudaError_t e = do_insert(f, resolve_insert(f, n), d_hashes, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "insert kernel launch");
}

static int find_common(const sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n, void* d_out,
                       bool bits, void* stream) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  if (n == 0) return SBBF_OK;
  if (!d_hashes || !d_out) return fail(SBBF_EINVAL, "null buffer");
  DeviceGuard g(f->di.device);
  sbbf_gpu* m = const_cast<sbbf_gpu*>(f);  // the blocked plan is created lazily
  cudaError_t e = do_find(m, resolve_find(f, n), d_hashes, n, d_out, bits, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "find kernel launch");
}

int sbbf_gpu_find_batch(const sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n,
                        uint8_t* d_results, void* stream) {
  return find_common(f, d_hashes, n, d_results, false, stream);
}

int sbbf_gpu_find_batch_bits(const sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n,
                             uint32_t* d_bits, void* stream) {
  return find_common(f, d_hashes, n, d_bits, true, stream);
}

int sbbf_gpu_add_hashes_host(sbbf_gpu_t* f, const uint64_t* h_hashes, uint64_t n) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  return host_pipeline(f, HostOp::kInsert, h_hashes, n, nullptr);
}

int sbbf_gpu_find_hashes_host(const sbbf_gpu_t* f, const uint64_t* h_hashes, uint64_t n,
                              uint8_t* h_results) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  return host_pipeline(const_cast<sbbf_gpu*>(f), HostOp::kFindBytes, h_hashes, n, h_results);
}

int sbbf_gpu_find_bits_host(const sbbf_gpu_t* f, const uint64_t* h_hashes, uint64_t n,
                            uint32_t* h_bits) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  return host_pipeline(const_cast<sbbf_gpu*>(f), HostOp::kFindBits, h_hashes, n, h_bits);
}

int sbbf_gpu_add_hash(sbbf_gpu_t* f, uint64_t hash) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  std::lock_guard<std::mutex> lock(f->host_mu);
  DeviceGuard g(f->di.device);
  // behind all queued work (as the host calls); the hash goes through the
  // pinned, device-mapped slot (no separate copy)
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) {
    f->h_one[0] = hash;
    e = sbbf::launch_insert(f->di, SBBF_INSERT_WIDE, f->d_blocks, f->geom, f->d_one, 1, nullptr);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "add_hash");
}

int sbbf_gpu_find_hash(const sbbf_gpu_t* f, uint64_t hash, int* found) {
  if (!f || !found) return fail(SBBF_EINVAL, "null argument");
  sbbf_gpu* m = const_cast<sbbf_gpu*>(f);
  std::lock_guard<std::mutex> lock(m->host_mu);
  DeviceGuard g(f->di.device);
  cudaError_t e = cudaDeviceSynchronize();  // behind all queued work, as the host calls
  if (e == cudaSuccess) {
    m->h_one[0] = hash;
    e = sbbf::launch_find(f->di, SBBF_FIND_GLOBAL, f->d_blocks, f->geom, m->d_one, 1, m->d_one + 1,
                          false, nullptr);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "find_hash");
  const uint8_t r = static_cast<uint8_t>(m->h_one[1] & 0xff);
  *found = r ? 1 : 0;
  return SBBF_OK;
}

int sbbf_gpu_to_host(const sbbf_gpu_t* f, void* h_dst, uint64_t bytes) {
  if (!f || !h_dst) return fail(SBBF_EINVAL, "null argument");
  if (bytes != f->nb * 32) return fail(SBBF_EINVAL, "bytes must equal num_buckets * 32");
  DeviceGuard g(f->di.device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(h_dst, f->d_blocks, bytes, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "to_host");
}

int sbbf_gpu_blocks_to_host(const sbbf_gpu_t* f, uint64_t first_block, uint64_t count,
                            void* h_dst) {
  if (!f || (count && !h_dst)) return fail(SBBF_EINVAL, "null argument");
  if (first_block > f->nb || count > f->nb - first_block)
    return fail(SBBF_EINVAL, "block range out of bounds");
  if (count == 0) return SBBF_OK;
  DeviceGuard g(f->di.device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(h_dst, f->d_blocks + first_block * 8, count * 32, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "blocks_to_host");
}

int sbbf_gpu_from_host(sbbf_gpu_t* f, const void* h_src, uint64_t bytes) {
  if (!f || !h_src) return fail(SBBF_EINVAL, "null argument");
  if (bytes != f->nb * 32) return fail(SBBF_EINVAL, "bytes must equal num_buckets * 32");
  DeviceGuard g(f->di.device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(f->d_blocks, h_src, bytes, cudaMemcpyHostToDevice);
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "from_host");
}

int sbbf_gpu_block_index_batch(const uint64_t* d_hashes, uint64_t n, uint64_t num_buckets,
                               uint64_t* d_out, void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_hashes || !d_out) return fail(SBBF_EINVAL, "null buffer");
  cudaError_t e = sbbf::launch_block_index(d_hashes, n, num_buckets, d_out,
                                           static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "block_index kernel");
}

int sbbf_gpu_make_mask_batch(const uint64_t* d_hashes, uint64_t n, uint32_t* d_lanes,
                             void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_hashes || !d_lanes) return fail(SBBF_EINVAL, "null buffer");
  cudaError_t e = sbbf::launch_make_mask(d_hashes, n, d_lanes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "make_mask kernel");
}

// Host-array forms of the two free functions (block_index filter.hpp:42,
// make_mask filter.hpp:47): the values are computed by the device kernels
// above on `device`, through a small device staging copy. For drop-in
// callers of the reference's free functions (tests/cpp/dropin/sbbf/filter.hpp).
namespace {
int host_free_fn(const uint64_t* h_hashes, uint64_t n, uint64_t num_buckets, void* h_out, size_t out_per_key,
                 bool mask, int device) {
  if (n == 0) return SBBF_OK;
  if (!h_hashes || !h_out) return fail(SBBF_EINVAL, "null buffer");
  if (device < 0 || device >= 64) return fail(SBBF_ENODEV, "bad device ordinal");
  DeviceGuard g(device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  // per-device staging, grown on demand and kept (these are called per value
  // by reference-style callers)
  static std::mutex mu;
  static uint64_t* d_buf[64] = {};
  static uint64_t cap[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  const uint64_t need = n * (sizeof(uint64_t) + out_per_key);
  cudaError_t e = cudaSuccess;
  if (cap[device] < need) {
    if (d_buf[device]) cudaFree(d_buf[device]);
    d_buf[device] = nullptr;
    cap[device] = 0;
    e = cudaMalloc(&d_buf[device], need);
    if (e == cudaSuccess) cap[device] = need;
  }
  uint64_t* d_in = d_buf[device];
  void* d_out = d_in + n;
  if (e == cudaSuccess) e = cudaMemcpy(d_in, h_hashes, n * sizeof(uint64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = mask ? sbbf::launch_make_mask(d_in, n, static_cast<uint32_t*>(d_out), nullptr)
             : sbbf::launch_block_index(d_in, n, num_buckets, static_cast<uint64_t*>(d_out), nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(h_out, d_out, n * out_per_key, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, mask ? "make_mask" : "block_index");
}
}  // namespace

int sbbf_gpu_block_index_host(const uint64_t* h_hashes, uint64_t n, uint64_t num_buckets, uint64_t* h_out,
                              int device) {
  if (num_buckets == 0) return fail(SBBF_EINVAL, "num_buckets must be >= 1");
  return host_free_fn(h_hashes, n, num_buckets, h_out, sizeof(uint64_t), false, device);
}

int sbbf_gpu_make_mask_host(const uint64_t* h_hashes, uint64_t n, uint32_t* h_lanes, int device) {
  return host_free_fn(h_hashes, n, 0, h_lanes, 8 * sizeof(uint32_t), true, device);
}

int sbbf_gpu_set_l2_fetch_granularity(int device, int bytes, int* old) {
  if (bytes < 0 || bytes > 128) return fail(SBBF_EINVAL, "granularity must be 0..128 bytes");
  DeviceGuard g(device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  size_t prev = 0;
  cudaError_t e = cudaDeviceGetLimit(&prev, cudaLimitMaxL2FetchGranularity);
  if (e == cudaSuccess) e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(bytes));
  if (e != cudaSuccess) return cuda_fail(e, "cudaLimitMaxL2FetchGranularity");
  if (old) *old = static_cast<int>(prev);
  return SBBF_OK;
}

int sbbf_gpu_release_scratch(sbbf_gpu_t* f) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  DeviceGuard g(f->di.device);
  std::lock_guard<std::mutex> lock(f->plan_mu);
  sbbf::blocked_ctx_release(f->plan.ctx);
  return SBBF_OK;
}

int sbbf_gpu_set_insert_variant(sbbf_gpu_t* f, int variant) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  if (variant < SBBF_INSERT_AUTO || variant > SBBF_INSERT_BLOCKED)
    return fail(SBBF_EINVAL, "unknown insert variant");
  f->insert_variant = variant;
  return SBBF_OK;
}

int sbbf_gpu_set_find_variant(sbbf_gpu_t* f, int variant) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  if (variant < SBBF_FIND_AUTO || variant > SBBF_FIND_BLOCKED)
    return fail(SBBF_EINVAL, "unknown find variant");
  if (variant == SBBF_FIND_SMEM && !smem_fits(f))
    return fail(SBBF_EINVAL, "filter too large for the shared-memory path");
  f->find_variant = variant;
  return SBBF_OK;
}

int sbbf_gpu_resolved_insert_variant(const sbbf_gpu_t* f, uint64_t n) {
  return f ? resolve_insert(f, n) : SBBF_EINVAL;
}

int sbbf_gpu_resolved_find_variant(const sbbf_gpu_t* f, uint64_t n) {
  return f ? resolve_find(f, n) : SBBF_EINVAL;
}

// ---- FilterImage v1 (persist.hpp:14-31, persist.cpp:72-157) -----------------
static void image_header(uint8_t hdr[17], uint64_t nb, uint32_t hasher_id) {
  hdr[0] = 'S';
  hdr[1] = 'B';
  hdr[2] = 'B';
  hdr[3] = 'F';
  hdr[4] = 1;  // kImageVersion, persist.hpp:21
  for (int i = 0; i < 4; ++i) hdr[5 + i] = static_cast<uint8_t>(hasher_id >> (8 * i));
  for (int i = 0; i < 8; ++i) hdr[9 + i] = static_cast<uint8_t>(nb >> (8 * i));
}

uint64_t sbbf_gpu_image_size(uint64_t num_buckets) { return 17 + 32 * num_buckets + 4; }

int sbbf_gpu_image_crc(const sbbf_gpu_t* f, uint32_t* crc) {
  if (!f || !crc) return fail(SBBF_EINVAL, "null argument");
  DeviceGuard g(f->di.device);
  uint8_t hdr[17];
  image_header(hdr, f->nb, f->hasher_id);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t body = 0;
  if (e == cudaSuccess) e = sbbf::device_crc32(f->d_blocks, f->nb * 32, &body, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "image crc");
  *crc = sbbf::crc32_combine(sbbf::crc32_host_update(0, hdr, 17), body, f->nb * 32);
  return SBBF_OK;
}

int sbbf_gpu_blocks_crc(const sbbf_gpu_t* f, uint32_t* crc) {
  if (!f || !crc) return fail(SBBF_EINVAL, "null argument");
  DeviceGuard g(f->di.device);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t body = 0;
  if (e == cudaSuccess) e = sbbf::device_crc32(f->d_blocks, f->nb * 32, &body, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "blocks crc");
  *crc = body;
  return SBBF_OK;
}

uint32_t sbbf_crc32_update(uint32_t crc, const void* data, uint64_t len) {
  return data ? sbbf::crc32_host_update(crc, static_cast<const uint8_t*>(data), len) : crc;
}

uint32_t sbbf_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
  return sbbf::crc32_combine(crc1, crc2, len2);
}

int sbbf_gpu_serialize(const sbbf_gpu_t* f, void* h_dst, uint64_t cap, uint64_t* written) {
  if (!f || !h_dst) return fail(SBBF_EINVAL, "null argument");
  const uint64_t size = sbbf_gpu_image_size(f->nb);
  if (cap < size) return fail(SBBF_EINVAL, "destination smaller than the image");
  uint8_t* out = static_cast<uint8_t*>(h_dst);
  image_header(out, f->nb, f->hasher_id);
  int rc = sbbf_gpu_to_host(f, out + 17, f->nb * 32);  // lanes are little-endian in HBM already
  uint32_t crc = 0;
  if (rc == SBBF_OK) rc = sbbf_gpu_image_crc(f, &crc);
  if (rc != SBBF_OK) return rc;
  for (int i = 0; i < 4; ++i) out[size - 4 + i] = static_cast<uint8_t>(crc >> (8 * i));
  if (written) *written = size;
  return SBBF_OK;
}

static uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// persist.cpp:90-126: same checks, same order, same codes (errc = 1 + PersistErrc).
int sbbf_gpu_deserialize(const void* h_img, uint64_t len, int device, sbbf_gpu_t** out, int* errc) {
  if (!out) return fail(SBBF_EINVAL, "out is null");
  *out = nullptr;
  auto bad = [&](int code, const char* msg) {
    if (errc) *errc = code;
    return fail(SBBF_EFORMAT, msg);
  };
  if (errc) *errc = 0;
  const uint8_t* b = static_cast<const uint8_t*>(h_img);
  if (!b || len < 21) return bad(1, "filter image shorter than fixed fields");
  if (b[0] != 'S' || b[1] != 'B' || b[2] != 'B' || b[3] != 'F') return bad(2, "not a filter image (bad magic)");
  if (b[4] != 1) return bad(3, "unsupported filter image version");
  const uint32_t hid = static_cast<uint32_t>(get_le(b + 5, 4));
  const uint64_t nb = get_le(b + 9, 8);
  if (nb == 0) return bad(4, "filter image declares zero buckets");
  if (nb > (~uint64_t{0} - 21) / 32 || len != sbbf_gpu_image_size(nb))
    return bad(1, "filter image length does not match its bucket count");
  sbbf_gpu_t* f = nullptr;
  int rc = sbbf_gpu_create(nb, device, &f);
  if (rc != SBBF_OK) return rc;
  rc = sbbf_gpu_from_host(f, b + 17, nb * 32);
  if (rc == SBBF_OK) rc = sbbf_gpu_set_hasher_id(f, hid);
  uint32_t crc = 0;
  if (rc == SBBF_OK) rc = sbbf_gpu_image_crc(f, &crc);
  if (rc != SBBF_OK) {
    sbbf_gpu_destroy(f);
    return rc;
  }
  if (crc != static_cast<uint32_t>(get_le(b + len - 4, 4))) {
    sbbf_gpu_destroy(f);
    return bad(5, "filter image checksum mismatch");
  }
  *out = f;
  return SBBF_OK;
}

// save_filter / load_filter (persist.cpp:128-157); I/O failures -> errc 6 (kIo).
int sbbf_gpu_save(const sbbf_gpu_t* f, const char* path, int* errc) {
  if (!f || !path) return fail(SBBF_EINVAL, "null argument");
  if (errc) *errc = 0;
  std::vector<uint8_t> img(sbbf_gpu_image_size(f->nb));
  int rc = sbbf_gpu_serialize(f, img.data(), img.size(), nullptr);
  if (rc != SBBF_OK) return rc;
  FILE* fp = std::fopen(path, "wb");
  const bool ok = fp && std::fwrite(img.data(), 1, img.size(), fp) == img.size() && std::fflush(fp) == 0;
  if (fp) std::fclose(fp);
  if (!ok) {
    if (errc) *errc = 6;
    return fail(SBBF_EFORMAT, std::string("cannot write ") + path);
  }
  return SBBF_OK;
}

int sbbf_gpu_load(const char* path, int device, sbbf_gpu_t** out, int* errc) {
  if (!path || !out) return fail(SBBF_EINVAL, "null argument");
  *out = nullptr;
  FILE* fp = std::fopen(path, "rb");
  if (!fp) {
    if (errc) *errc = 6;
    return fail(SBBF_EFORMAT, std::string("cannot open ") + path);
  }
  std::vector<uint8_t> bytes;
  uint8_t chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof(chunk), fp)) > 0) bytes.insert(bytes.end(), chunk, chunk + got);
  const bool err = std::ferror(fp) != 0;
  std::fclose(fp);
  if (err) {
    if (errc) *errc = 6;
    return fail(SBBF_EFORMAT, std::string("read failed for ") + path);
  }
  return sbbf_gpu_deserialize(bytes.data(), bytes.size(), device, out, errc);
}

// ---- XXH64 key frontend (hash.hpp:11-25, hash.cpp:100-114) -----------------
int sbbf_gpu_hash_u64_keys(const uint64_t* d_keys, uint64_t n, uint64_t seed, uint64_t* d_hashes,
                           void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_keys || !d_hashes) return fail(SBBF_EINVAL, "null buffer");
  cudaError_t e = sbbf::launch_hash_u64(d_keys, n, seed, d_hashes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "hash kernel");
}

int sbbf_gpu_hash_bytes(const uint8_t* d_data, const uint64_t* d_offsets, uint64_t n, uint64_t seed,
                        uint64_t* d_hashes, void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_offsets || !d_hashes) return fail(SBBF_EINVAL, "null buffer");
  cudaError_t e =
      sbbf::launch_hash_bytes(d_data, d_offsets, n, seed, d_hashes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "hash kernel");
}

int sbbf_gpu_hash_counter_strings(uint64_t start, uint64_t n, uint64_t seed, uint64_t* d_hashes, void* stream) {
  if (n == 0) return SBBF_OK;
  if (!d_hashes) return fail(SBBF_EINVAL, "null buffer");
  cudaError_t e = sbbf::launch_hash_decimal(start, n, seed, d_hashes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "hash kernel");
}

// Hash-then-dispatch for the paths without a fused kernel (blocked, forced
// variants): the hashes go to stream-ordered scratch.
static cudaError_t with_hashed(const uint64_t* keys, uint64_t n, uint64_t seed, cudaStream_t s,
                               const std::function<cudaError_t(const uint64_t*)>& body) {
  uint64_t* tmp = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * sizeof(uint64_t), s);
  if (e == cudaSuccess) e = sbbf::launch_hash_u64(keys, n, seed, tmp, s);
  if (e == cudaSuccess) e = body(tmp);
  if (tmp) cudaFreeAsync(tmp, s);
  return e;
}

int sbbf_gpu_insert_keys_u64(sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                             void* stream) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  if (n == 0) return SBBF_OK;
  if (!d_keys) return fail(SBBF_EINVAL, "null keys");
  DeviceGuard g(f->di.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int v = resolve_insert(f, n);
  cudaError_t e;
  if (v == SBBF_INSERT_WIDE || v == SBBF_INSERT_WIDE_TEST)
    e = sbbf::launch_insert_keys(f->di, v == SBBF_INSERT_WIDE_TEST, f->d_blocks, f->geom, d_keys, n, seed, s);
  else
    e = with_hashed(d_keys, n, seed, s, [&](const uint64_t* h) { return do_insert(f, v, h, n, s); });
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "insert_keys");
}

static int find_keys_common(const sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                            void* d_out, bool bits, void* stream) {
  if (!f) return fail(SBBF_EINVAL, "null filter");
  if (n == 0) return SBBF_OK;
  if (!d_keys || !d_out) return fail(SBBF_EINVAL, "null buffer");
  DeviceGuard g(f->di.device);
  sbbf_gpu* m = const_cast<sbbf_gpu*>(f);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int v = resolve_find(f, n);
  cudaError_t e;
  if (v == SBBF_FIND_GLOBAL)
    e = sbbf::launch_find_keys(f->di, f->d_blocks, f->geom, d_keys, n, seed, d_out, bits, s);
  else
    e = with_hashed(d_keys, n, seed, s, [&](const uint64_t* h) { return do_find(m, v, h, n, d_out, bits, s); });
  return e == cudaSuccess ? SBBF_OK : cuda_fail(e, "find_keys");
}

int sbbf_gpu_find_keys_u64(const sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                           uint8_t* d_results, void* stream) {
  return find_keys_common(f, d_keys, n, seed, d_results, false, stream);
}

int sbbf_gpu_find_keys_u64_bits(const sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                                uint32_t* d_bits, void* stream) {
  return find_keys_common(f, d_keys, n, seed, d_bits, true, stream);
}

}  // extern "C"
