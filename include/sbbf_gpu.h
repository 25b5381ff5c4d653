/*
 * sbbf_gpu.h — C ABI of the B200-native split block Bloom filter.
 *
 * Drop-in for the batched build/probe path of the reference core
 * (/root/reference/proj/core/include/sbbf/filter.hpp, class
 * sbbf::SplitBlockFilter). Each entry point below names the reference
 * interface it replaces (file:line, relative to /root/reference/proj/).
 *
 * Bit layout is the reference's exactly (filter.hpp:11-31): an array of
 * num_buckets 32-byte blocks, eight little-endian 32-bit lanes each, lane 0
 * lowest-addressed. block_index = floor(hash * num_buckets / 2^64)
 * (filter.cpp:125-127); lane i's bit = (seed_i * low32(hash)) >> 27
 * (filter.cpp:129-138). A filter built here is byte-identical to the
 * reference's for the same hashes in any order.
 *
 * Conventions
 *  - Every function returns SBBF_OK (0) or a negative SBBF_E* code; no C++
 *    exception crosses the ABI. sbbf_gpu_last_error() returns a
 *    thread-local message for the most recent failure on this thread.
 *  - "d_" pointers are device pointers on the filter's device, owned by the
 *    caller. "h_" pointers are host pointers (pinned or pageable).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream). Device-pointer operations are asynchronous and stream-ordered.
 *    Host-pointer operations (*_host, add_hash/find_hash) and
 *    to_host/from_host are synchronous and start behind ALL work already
 *    queued on the filter's device (cudaDeviceSynchronize first), so device
 *    inserts queued on any stream are visible to a following host lookup.
 *  - Lookups are launched as programmatic dependents of the previous grid on
 *    the stream (PDL). They read nothing — neither the filter nor the
 *    caller's hashes — before griddepcontrol.wait, so the hashes may come
 *    from the kernel launched just before (e.g. a hashing kernel).
 *  - Inserts use atomic OR (red.global.or), so concurrent insert_batch calls
 *    on one handle are safe — the "atomic OR writes" option SPEC.md:131
 *    permits. A find concurrent with an insert may see either answer for
 *    in-flight keys (bits are monotone).
 *  - There is no CPU fallback: without a usable CUDA device, create() fails
 *    with SBBF_ENODEV.
 */
#ifndef SBBF_GPU_H
#define SBBF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is the only exported surface */
#endif

#define SBBF_GPU_ABI_VERSION 1

enum {
  SBBF_OK = 0,
  SBBF_EINVAL = -1,  /* bad argument; num_buckets == 0 mirrors std::invalid_argument (filter.cpp:160-162) */
  SBBF_ENOMEM = -2,  /* device or host allocation failed ("resource error") */
  SBBF_ECUDA = -3,   /* any other CUDA runtime error */
  SBBF_ENODEV = -4,  /* no CUDA device / bad device ordinal */
  SBBF_EFORMAT = -5  /* FilterImage parse failure */
};

/* Insert strategies (sbbf_gpu_set_insert_variant). AUTO picks per call. */
enum {
  SBBF_INSERT_AUTO = 0,
  SBBF_INSERT_LANE8 = 1,      /* 8 threads per key, one red.or per lane: 1 sector op / key */
  SBBF_INSERT_LANE8_TEST = 2, /* as LANE8, but skip lanes whose bit is already set (hot keys) */
  SBBF_INSERT_THREAD = 3,     /* 1 thread per key, 8 red.or per key (baseline variant) */
  SBBF_INSERT_WIDE = 4,       /* 4 threads per key, one 64-bit red.or per lane pair */
  SBBF_INSERT_WIDE_TEST = 5,  /* as WIDE, skipping lane pairs whose bits are all set */
  SBBF_INSERT_BLOCKED = 6     /* group the batch by filter slice first, then insert slice by
                                 slice so the atomics hit L2 (filters beyond L2) */
};

/* Lookup strategies (sbbf_gpu_set_find_variant). AUTO picks per call. */
enum {
  SBBF_FIND_AUTO = 0,
  SBBF_FIND_GLOBAL = 1, /* one 256-bit LDG per key from L2/HBM */
  SBBF_FIND_SMEM = 2,   /* filter staged into shared memory per CTA (small filters only) */
  SBBF_FIND_BLOCKED = 3 /* group the batch by filter slice, probe slice by slice from L2 */
};

typedef struct sbbf_gpu sbbf_gpu_t;

/* --- lifetime: SplitBlockFilter(num_buckets, hasher_id, backend)
 *     filter.hpp:67-71, filter.cpp:148-163 ----------------------------- */
/* Allocates a zeroed, 256-byte-aligned block array of num_buckets*32 bytes on
 * `device`. SBBF_EINVAL if num_buckets == 0. */
int sbbf_gpu_create(uint64_t num_buckets, int device, sbbf_gpu_t** out);
int sbbf_gpu_destroy(sbbf_gpu_t* f);
/* Zero every block (stream-ordered). Equivalent to a fresh filter. */
int sbbf_gpu_clear(sbbf_gpu_t* f, void* stream);

/* --- accessors: filter.hpp:85-94 -------------------------------------- */
uint64_t sbbf_gpu_num_buckets(const sbbf_gpu_t* f);
uint64_t sbbf_gpu_size_bytes(const sbbf_gpu_t* f);
uint32_t sbbf_gpu_hasher_id(const sbbf_gpu_t* f);
int sbbf_gpu_set_hasher_id(sbbf_gpu_t* f, uint32_t hasher_id);
int sbbf_gpu_device(const sbbf_gpu_t* f);
/* Raw device pointer to the block array (num_buckets*32 bytes). */
void* sbbf_gpu_device_blocks(sbbf_gpu_t* f);

/* --- batched hot path: add_hashes / find_hashes, filter.hpp:81-83,
 *     filter.cpp:184-207 ---------------------------------------------- */
int sbbf_gpu_insert_batch(sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n, void* stream);
/* results[k] = 1 if hashes[k] may be present else 0, one byte per key,
 * identical to the reference's `results` (filter.cpp:91). */
int sbbf_gpu_find_batch(const sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n,
                        uint8_t* d_results, void* stream);
/* Packed lookup bitmap: bit (k % 32) of word k / 32 is key k (LSB-first);
 * bits past n in the last word are 0. d_bits holds ceil(n/32) words. */
int sbbf_gpu_find_batch_bits(const sbbf_gpu_t* f, const uint64_t* d_hashes, uint64_t n,
                             uint32_t* d_bits, void* stream);

/* --- host-buffer drop-ins: add_hashes(span) / find_hashes(span, uint8_t*)
 *     with the caller's host memory, filter.hpp:81-83. Chunked, with the
 *     host<->device copies overlapped with the kernels on three streams.
 *     Synchronous on return. ------------------------------------------ */
int sbbf_gpu_add_hashes_host(sbbf_gpu_t* f, const uint64_t* h_hashes, uint64_t n);
int sbbf_gpu_find_hashes_host(const sbbf_gpu_t* f, const uint64_t* h_hashes, uint64_t n,
                              uint8_t* h_results);
int sbbf_gpu_find_bits_host(const sbbf_gpu_t* f, const uint64_t* h_hashes, uint64_t n,
                            uint32_t* h_bits);

/* --- single-key ops: add_hash / find_hash, filter.hpp:77-78 (convenience;
 *     each is one launch + sync — use the batch calls for throughput). - */
int sbbf_gpu_add_hash(sbbf_gpu_t* f, uint64_t hash);
/* *found = 0/1 */
int sbbf_gpu_find_hash(const sbbf_gpu_t* f, uint64_t hash, int* found);

/* --- blocks() / from_blocks(): filter.hpp:74-75,87. Synchronous. ------ */
/* Copies exactly num_buckets*32 bytes (bytes must equal that). Waits for
 * all work on the device first. */
int sbbf_gpu_to_host(const sbbf_gpu_t* f, void* h_dst, uint64_t bytes);
/* Copies blocks [first_block, first_block + count) (count*32 bytes); for
 * spot checks of very large filters and for gathering shards. */
int sbbf_gpu_blocks_to_host(const sbbf_gpu_t* f, uint64_t first_block, uint64_t count,
                            void* h_dst);
/* Overwrites the block array from num_buckets*32 host bytes (adopts
 * existing contents, like from_blocks). */
int sbbf_gpu_from_host(sbbf_gpu_t* f, const void* h_src, uint64_t bytes);

/* --- free functions on device, for known-answer tests:
 *     block_index filter.hpp:42, make_mask filter.hpp:47 ---------------- */
int sbbf_gpu_block_index_batch(const uint64_t* d_hashes, uint64_t n, uint64_t num_buckets,
                               uint64_t* d_out, void* stream);
/* d_lanes holds n*8 uint32 (LaneMask per key, lane 0 first). */
int sbbf_gpu_make_mask_batch(const uint64_t* d_hashes, uint64_t n, uint32_t* d_lanes,
                             void* stream);

/* The same on host arrays (computed by the device kernels on `device`,
 * synchronous): what a caller of the reference's free functions links. */
int sbbf_gpu_block_index_host(const uint64_t* h_hashes, uint64_t n, uint64_t num_buckets, uint64_t* h_out,
                              int device);
int sbbf_gpu_make_mask_host(const uint64_t* h_hashes, uint64_t n, uint32_t* h_lanes, int device);

/* Filters beyond L2 keep the blocked path's scratch (about 11 B per key of
 * the largest batch chunk, up to ~6 GB for 2^28-key lookup rounds) cached on
 * the handle between calls; this returns it to the device (synchronous). */
int sbbf_gpu_release_scratch(sbbf_gpu_t* f);

/* --- tuning ----------------------------------------------------------- */
int sbbf_gpu_set_insert_variant(sbbf_gpu_t* f, int variant);
int sbbf_gpu_set_find_variant(sbbf_gpu_t* f, int variant);
/* Variant the AUTO policy would use for a batch of n keys (for reporting). */
int sbbf_gpu_resolved_insert_variant(const sbbf_gpu_t* f, uint64_t n);
int sbbf_gpu_resolved_find_variant(const sbbf_gpu_t* f, uint64_t n);

/* --- FilterImage v1: serialize / deserialize / save_filter / load_filter
 *     (persist.hpp:14-31,50-66; persist.cpp:72-157). The image is
 *     "SBBF" | version 1 | hasher id (u32 LE) | bucket count (u64 LE) |
 *     blocks | CRC-32 (IEEE) of everything before it. The CRC of the block
 *     array is computed on the GPU. Format errors return SBBF_EFORMAT with
 *     *errc = 1 + PersistErrc: 1 truncated, 2 bad magic, 3 bad version,
 *     4 zero buckets, 5 bad checksum, 6 I/O. --------------------------- */
uint64_t sbbf_gpu_image_size(uint64_t num_buckets);
int sbbf_gpu_image_crc(const sbbf_gpu_t* f, uint32_t* crc);
int sbbf_gpu_serialize(const sbbf_gpu_t* f, void* h_dst, uint64_t cap, uint64_t* written);
/* CRC-32 (IEEE, crc32_ieee persist.cpp:15-40) of the block array bytes alone,
 * computed on the GPU: a shard's contribution to the gathered image CRC. */
int sbbf_gpu_blocks_crc(const sbbf_gpu_t* f, uint32_t* crc);
/* Host CRC-32 helpers: continue `crc` over len bytes, and the CRC of A||B
 * from crc(A), crc(B) and len(B) (zlib's crc32_combine). Shards' block CRCs
 * combine in rank order into the gathered filter's image CRC without moving
 * the blocks. */
uint32_t sbbf_crc32_update(uint32_t crc, const void* data, uint64_t len);
uint32_t sbbf_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2);
int sbbf_gpu_deserialize(const void* h_img, uint64_t len, int device, sbbf_gpu_t** out, int* errc);
int sbbf_gpu_save(const sbbf_gpu_t* f, const char* path, int* errc);
int sbbf_gpu_load(const char* path, int device, sbbf_gpu_t** out, int* errc);

/* --- XXH64 key frontend: kHasherXxh64 (hash.hpp:12), hash_key /
 *     hash_u64_key (hash.hpp:20-25, hash.cpp:100-114) ----------------------
 * u64 keys hash as their 8 little-endian bytes; byte-string key i is
 * d_data[d_offsets[i], d_offsets[i+1]) (n+1 offsets). The *_keys_u64 calls
 * hash inside the insert / lookup kernel (no hash array in HBM); pair them
 * with sbbf_gpu_set_hasher_id(f, 1) so images record the frontend. */
int sbbf_gpu_hash_u64_keys(const uint64_t* d_keys, uint64_t n, uint64_t seed, uint64_t* d_hashes,
                           void* stream);
int sbbf_gpu_hash_bytes(const uint8_t* d_data, const uint64_t* d_offsets, uint64_t n, uint64_t seed,
                        uint64_t* d_hashes, void* stream);
/* hash_key(std::to_string(c), seed) for c = start .. start+n-1: the
 * reference's byte-string experiment keys (KeyMode::kByteStrings,
 * tools/harness.cpp:60-65), digits built on the device. */
int sbbf_gpu_hash_counter_strings(uint64_t start, uint64_t n, uint64_t seed, uint64_t* d_hashes, void* stream);
/* Monte-Carlo false-positive oracle (sbbf_fpp_mc, model.cpp:105-128) on the
 * GPU: `blocks` blocks each filled with Poisson(a) hashes from the block's
 * preimage interval, then `trials` uniform probes; *fpp = hits / trials.
 * Same distributions as the reference, counter-based per-block streams
 * (seed-reproducible, not the reference's mt19937_64 draws). Errors as the
 * reference's domain_error cases: a < 0, a > 500, blocks or trials == 0. */
int sbbf_gpu_fpp_mc(double a, uint64_t blocks, uint64_t trials, uint64_t seed, int device, double* fpp);
int sbbf_gpu_insert_keys_u64(sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                             void* stream);
int sbbf_gpu_find_keys_u64(const sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                           uint8_t* d_results, void* stream);
int sbbf_gpu_find_keys_u64_bits(const sbbf_gpu_t* f, const uint64_t* d_keys, uint64_t n, uint64_t seed,
                                uint32_t* d_bits, void* stream);

/* --- multi-GPU shards (no reference counterpart: the reference has no
 *     distributed mode) -----------------------------------
 * Rank r of P owns global blocks [floor(r*B/P), floor((r+1)*B/P)). A shard
 * keeps the global block_index (taken against total_buckets), so the shards
 * concatenated in rank order are byte-identical to one B-bucket filter.
 * Shard kernels ignore (insert) / answer 0 for (find) keys it does not own. */
int sbbf_gpu_create_shard(uint64_t total_buckets, uint64_t first_block, uint64_t num_buckets,
                          int device, sbbf_gpu_t** out);
uint64_t sbbf_gpu_total_buckets(const sbbf_gpu_t* f);
uint64_t sbbf_gpu_first_block(const sbbf_gpu_t* f);
/* h_bounds[0..parts] = floor(r * total_buckets / parts) (host). */
int sbbf_shard_bounds(uint64_t total_buckets, uint32_t parts, uint64_t* h_bounds);
/* d_counts[r] = number of keys whose block falls in shard r (parts <= 1024;
 * d_bounds = the first `parts` entries of sbbf_shard_bounds, on device). */
int sbbf_shard_count(const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                     const uint64_t* d_bounds, uint32_t parts, uint64_t* d_counts, void* stream);
/* Group keys by destination shard: segment r of d_out starts at d_offsets[r]
 * (exclusive prefix sum of the counts). d_pos (optional, n < 2^32) gets each
 * key's source index; d_cursor is parts u64 of scratch. Order inside a
 * segment is unspecified. */
int sbbf_shard_scatter(const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                       const uint64_t* d_bounds, uint32_t parts, const uint64_t* d_offsets,
                       uint64_t* d_cursor, uint64_t* d_out, uint32_t* d_pos, void* stream);
/* One call for count + scatter (parts <= 64): warp-ballot multisplit, shard
 * segments staged through shared memory for coalesced stores, no host sync.
 * d_counts[r] = keys for shard r; segment r of d_out starts at the exclusive
 * prefix sum of d_counts; d_scratch is parts u64. */
int sbbf_shard_partition(const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                         const uint64_t* d_bounds, uint32_t parts, uint64_t* d_counts, uint64_t* d_scratch,
                         uint64_t* d_out, uint32_t* d_pos, void* stream);
/* d_dst[d_pos[i]] = d_src[i]: lookup answers back to source order. */
int sbbf_scatter_u8(const uint8_t* d_src, const uint32_t* d_pos, uint64_t n, uint8_t* d_dst,
                    void* stream);
/* Pack 0/1 bytes into an LSB-first bitmap of ceil(n/32) words. */
int sbbf_pack_bits(const uint8_t* d_src, uint64_t n, uint32_t* d_bits, void* stream);

/* --- fused multi-GPU dispatch over peer memory (SURVEY.md §8(e) "fused
 *     option"; sbbf_route.cu) ---------------------------------------------
 * Each rank owns a receive window (one cudaMalloc, exported by CUDA IPC
 * handle) with a region per source rank and two parities. dispatch
 * partitions a batch by owner shard and the scatter stores each owner's run
 * straight into that owner's window over NVLink (no staging array, no
 * counts exchange, no host sync). Per collective call, every rank runs:
 *   insert: dispatch(keep_positions=0); barrier; insert_window
 *   lookup: dispatch(keep_positions=1); barrier; find_window; barrier; combine
 * where "barrier" is any stream-ordered collective (e.g. a 1-element NCCL
 * all-reduce). Batches are <= max_batch keys per rank per call. */
typedef struct sbbf_route sbbf_route_t;
uint64_t sbbf_route_window_bytes(uint32_t parts, uint64_t max_batch);
int sbbf_route_create(uint32_t parts, uint32_t rank, uint64_t max_batch, int device, sbbf_route_t** out);
void sbbf_route_destroy(sbbf_route_t* rt);
uint64_t sbbf_route_max_batch(const sbbf_route_t* rt);
/* 64-byte CUDA IPC handle of this rank's window (exchange it out of band). */
int sbbf_route_ipc_handle(const sbbf_route_t* rt, void* handle);
/* Map peer `peer`'s window from its handle (another process). */
int sbbf_route_open_peer(sbbf_route_t* rt, uint32_t peer, const void* handle);
/* Same-process link (P shards driven by one process, e.g. tests). */
int sbbf_route_link_local(sbbf_route_t* rt, uint32_t peer, const sbbf_route_t* other);
int sbbf_route_ready(const sbbf_route_t* rt);
int sbbf_route_dispatch(sbbf_route_t* rt, const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                        const uint64_t* d_bounds, int keep_positions, void* stream);
int sbbf_route_insert_window(sbbf_route_t* rt, sbbf_gpu_t* shard, void* stream);
int sbbf_route_find_window(sbbf_route_t* rt, const sbbf_gpu_t* shard, void* stream);
/* d_results[i] = answer for key i of the last lookup dispatch (0/1 bytes). */
int sbbf_route_combine(sbbf_route_t* rt, uint8_t* d_results, void* stream);

/* --- multi-GPU sharded filter (SURVEY.md §8(b) "sharded layer") ----------
 * One rank per GPU of an NCCL communicator (ncclComm_t passed as void*).
 * Rank r owns blocks [floor(rB/P), floor((r+1)B/P)) and routes keys through
 * the fused peer-memory dispatch above; the phases are ordered by 1-element
 * NCCL all-reduces on the caller's stream (no host sync). insert / find /
 * find_bits are collective (every rank calls them, batches <= max_batch
 * keys per rank); any rank may pass any keys. NCCL is loaded at run time
 * (libnccl.so.2): without it these return SBBF_ENODEV. */
typedef struct sbbf_dist sbbf_dist_t;
/* 128-byte ncclUniqueId from rank 0, to broadcast out of band, and a
 * communicator built from it (for callers without one). */
int sbbf_dist_unique_id(void* id);
int sbbf_dist_comm_init(const void* id, int world, int rank, int device, void** comm);
int sbbf_dist_comm_destroy(void* comm);
int sbbf_dist_create(void* comm, uint64_t total_buckets, uint64_t max_batch, int device, sbbf_dist_t** out);
int sbbf_dist_destroy(sbbf_dist_t* d);
int sbbf_dist_rank(const sbbf_dist_t* d);
int sbbf_dist_world(const sbbf_dist_t* d);
/* This rank's shard (a filter handle: blocks, image CRC, ...). */
sbbf_gpu_t* sbbf_dist_shard(sbbf_dist_t* d);
int sbbf_dist_insert(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, void* stream);
int sbbf_dist_find(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, uint8_t* d_results, void* stream);
int sbbf_dist_find_bits(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, uint32_t* d_bits, void* stream);
/* Whole filter into h_dst (total_buckets*32 bytes) on rank `root`. */
int sbbf_dist_gather(sbbf_dist_t* d, void* h_dst, int root);
/* FilterImage CRC of the gathered filter (shard CRCs on each GPU, combined in
 * rank order; no block movement). Collective; every rank gets it. */
int sbbf_dist_image_crc(sbbf_dist_t* d, uint32_t* crc);
/* Failure detection: wait for `stream` on the host while polling
 * ncclCommGetAsyncError. On an asynchronous NCCL error (a dead peer, a
 * network fault) or after timeout_ms (<= 0: no deadline) the communicator is
 * aborted (ncclCommAbort, which also frees it: the caller must not destroy
 * that communicator afterwards), the call returns SBBF_ECUDA and every later
 * call on the handle fails fast instead of hanging in a barrier. */
int sbbf_dist_sync(sbbf_dist_t* d, void* stream, int64_t timeout_ms);
/* The same layer over caller-provided collectives instead of NCCL (e.g. a
 * host process group, or one GPU shared by several processes, which NCCL
 * refuses). allgather: rank-order gather of `bytes` host bytes from every
 * rank into recv (world*bytes). barrier: every rank's work queued on its
 * stream before the call completes before any rank's work queued after it
 * (may synchronize the stream on the host). Both return 0 on success. */
typedef struct sbbf_dist_hooks {
  int rank, world;
  void* ctx;
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes);
  int (*barrier)(void* ctx, void* stream);
} sbbf_dist_hooks;
int sbbf_dist_create_hooks(const sbbf_dist_hooks* hooks, uint64_t total_buckets, uint64_t max_batch, int device,
                           sbbf_dist_t** out);

/* L2 fetch-granularity hint for `device` (cudaLimitMaxL2FetchGranularity,
 * 0..128 bytes; process-wide for that device). 32 makes a random 32-byte
 * block miss fetch one sector from HBM instead of a wider line. *old (if
 * non-NULL) receives the previous value. */
int sbbf_gpu_set_l2_fetch_granularity(int device, int bytes, int* old);

/* --- diagnostics ------------------------------------------------------ */
const char* sbbf_gpu_last_error(void);
int sbbf_gpu_abi_version(void);
/* Number of kernels this library has launched in this process (all
 * devices); bench.py reports the delta over the timed region. */
uint64_t sbbf_gpu_launch_count(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* SBBF_GPU_H */
