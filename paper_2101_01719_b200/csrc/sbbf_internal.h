// sbbf_internal.h — launchers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "sbbf_bench.h"
#include "sbbf_gpu.h"
#include "sbbf_workload.h"

namespace sbbf {

struct DeviceInfo {
  int device = 0;
  int sms = 148;
  size_t smem_optin = 227 * 1024;  // cudaDevAttrMaxSharedMemoryPerBlockOptin
  size_t l2_bytes = 126u << 20;
};

// Filter geometry: block_index is taken against nb_global (the whole
// filter's bucket count), then offset by the shard's first block. A
// single-GPU filter is the shard {nb, 0, nb}.
struct Geom {
  uint64_t nb_global;
  uint64_t first;
  uint64_t nb_local;
};

constexpr int kInsertLane8 = SBBF_INSERT_LANE8;
constexpr int kInsertLane8Test = SBBF_INSERT_LANE8_TEST;
constexpr int kInsertThread = SBBF_INSERT_THREAD;
constexpr int kInsertWide = SBBF_INSERT_WIDE;
constexpr int kInsertWideTest = SBBF_INSERT_WIDE_TEST;
constexpr int kFindGlobal = SBBF_FIND_GLOBAL;
constexpr int kFindSmem = SBBF_FIND_SMEM;

uint64_t launch_count();
void set_last_error(const std::string& msg);  // what sbbf_gpu_last_error() returns on this thread
void note_launch();
uint64_t grid_for(uint64_t work_items, uint64_t items_per_block, int sms, int per_sm);

// 0, or k for 2^k range-split passes of the direct insert / lookup over a whole
// filter somewhat larger than L2 (sbbf_kernels.cu).
int split_log2(const DeviceInfo& di, const Geom& g, bool lookup);

cudaError_t launch_insert(const DeviceInfo& di, int variant, uint32_t* blocks, const Geom& g,
                          const uint64_t* hashes, uint64_t n, cudaStream_t s);
cudaError_t launch_find(const DeviceInfo& di, int variant, const uint32_t* blocks, const Geom& g,
                        const uint64_t* hashes, uint64_t n, void* out, bool bits, cudaStream_t s);
// Bucket `hashes` by block range: bucket k holds the keys whose block_index
// (against `total`) lies in [d_bounds[k], d_bounds[k+1]). Writes the counts,
// their exclusive prefix sum, the grouped keys and (optionally) each key's
// source index. All stream-ordered, no host sync. parts <= 1024.
cudaError_t launch_partition(const uint64_t* hashes, uint64_t n, uint64_t total, const uint64_t* d_bounds,
                             uint32_t parts, uint64_t* d_counts, uint64_t* d_offsets, uint64_t* d_cursor,
                             uint64_t* d_out, uint32_t* d_pos, int sms, cudaStream_t s);

// Group keys by owning shard (parts <= 64, exact ranges d_bounds[0..parts)):
// ballot-multisplit count + scan + shared-memory-staged scatter, no host
// sync. d_counts receives the per-shard counts; d_cursor is scratch.
cudaError_t shard_partition(const DeviceInfo& di, uint64_t total, uint32_t parts, const uint64_t* d_bounds,
                            const uint64_t* hashes, uint64_t n, uint64_t* d_counts, uint64_t* d_cursor,
                            uint64_t* d_out, uint32_t* d_pos, cudaStream_t s);

// Fused dispatch (sbbf_route.cu): the shard partition whose scatter writes
// bucket b's run straight to d_dst[b][0..count) — destination b's receive
// window, a peer GPU's memory mapped over NVLink — and stores the count at
// *d_count_dst[b]. d_counts receives the per-destination counts locally,
// d_pos (optional) the source index of every routed slot (bucket-major).
cudaError_t route_partition(const DeviceInfo& di, uint64_t total, uint32_t parts, const uint64_t* d_bounds,
                            const uint64_t* hashes, uint64_t n, uint64_t* d_counts, uint32_t* d_pos,
                            uint64_t* const* d_dst, unsigned long long* const* d_count_dst, cudaStream_t s);

// insert_wide over `n` keys with one warp step per 128 keys and the grid
// covering the batch once, so CTAs run in key order (blocked path).
cudaError_t launch_insert_ordered(const DeviceInfo& di, uint32_t* blocks, const Geom& g,
                                  const uint64_t* hashes, uint64_t n, bool test, cudaStream_t s);

// L2-blocked paths for filters larger than L2 (sbbf_blocked.cu).
struct BlockedCtx;  // per-handle scratch arena + side stream (sbbf_blocked.cu)
BlockedCtx* blocked_ctx_create();
void blocked_ctx_destroy(BlockedCtx* c);
int blocked_ctx_release(BlockedCtx* c);  // frees the arena (waits for its last use)
struct BlockedPlan {
  BlockedCtx* ctx = nullptr;      // null: per-call pool scratch
  uint32_t parts = 0;             // filter slices (per super-slice when super_parts > 1)
  const uint64_t* d_bounds = nullptr;  // parts entries, global block ids
  // Filters beyond 64 slices: super_parts exact block ranges, each blocked on
  // its own (two-level path). Bounds are local block ids; the host copy has
  // super_parts + 1 entries (the last = the shard's block count).
  uint32_t super_parts = 1;
  const uint64_t* d_super_bounds = nullptr;
  std::vector<uint64_t> h_super_bounds;
};
cudaError_t blocked_insert(const DeviceInfo& di, uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                           const uint64_t* hashes, uint64_t n, cudaStream_t s);
// dense_only (AUTO dispatch): the fused lookup sweep only for batches of at
// least a key per block; an explicit SBBF_FIND_BLOCKED takes it whenever the
// slices pack.
cudaError_t blocked_find(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                         const uint64_t* hashes, uint64_t n, void* out, bool bits, cudaStream_t s,
                         bool dense_only = false);

// The same over several key arrays at once (a rank's receive-window
// regions): one filter sweep, no staging copy. cudaErrorNotSupported when
// the plan is two-level or the regions exceed one blocked round.
cudaError_t blocked_insert_regions(const DeviceInfo& di, uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                                   const uint64_t* const* keys, const uint64_t* counts, uint32_t nr, cudaStream_t s);
cudaError_t blocked_find_regions(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const BlockedPlan& plan,
                                 const uint64_t* const* keys, const uint64_t* counts, uint32_t nr, uint8_t* const* outs,
                                 cudaStream_t s, bool dense_only = false);

// Filter-handle entry points for the route layer (sbbf_capi.cu): the blocked
// region path when AUTO would block the gathered batch; *handled = false
// otherwise (the caller gathers and uses the public ABI).
int gpu_insert_regions(sbbf_gpu_t* f, const uint64_t* const* keys, const uint64_t* counts, uint32_t nr,
                       cudaStream_t s, bool* handled);
int gpu_find_regions(const sbbf_gpu_t* f, const uint64_t* const* keys, const uint64_t* counts, uint32_t nr,
                     uint8_t* const* outs, cudaStream_t s, bool* handled);

// XXH64 key frontend (kHasherXxh64): hashing kernels and fused insert/find.
cudaError_t launch_hash_u64(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out, cudaStream_t s);
cudaError_t launch_hash_bytes(const uint8_t* data, const uint64_t* offsets, uint64_t n, uint64_t seed,
                              uint64_t* out, cudaStream_t s);
cudaError_t launch_hash_decimal(uint64_t start, uint64_t n, uint64_t seed, uint64_t* out, cudaStream_t s);
cudaError_t launch_insert_keys(const DeviceInfo& di, bool test, uint32_t* blocks, const Geom& g,
                               const uint64_t* keys, uint64_t n, uint64_t seed, cudaStream_t s);
cudaError_t launch_find_keys(const DeviceInfo& di, const uint32_t* blocks, const Geom& g, const uint64_t* keys,
                             uint64_t n, uint64_t seed, void* out, bool bits, cudaStream_t s);

// FilterImage CRC-32 (sbbf_image.cu): standard CRC-32 of `bytes` device
// bytes (synchronises `s`), and host helpers to extend / combine CRCs.
cudaError_t device_crc32(const void* d_data, uint64_t bytes, uint32_t* crc_out, cudaStream_t s);
uint32_t crc32_host_update(uint32_t crc, const uint8_t* p, uint64_t n);
uint32_t crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2);

cudaError_t launch_block_index(const uint64_t* h, uint64_t n, uint64_t nb, uint64_t* out,
                               cudaStream_t s);
cudaError_t launch_make_mask(const uint64_t* h, uint64_t n, uint32_t* out, cudaStream_t s);

}  // namespace sbbf
