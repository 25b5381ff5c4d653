// sbbf_dist.cu — the multi-GPU sharded filter as a C ABI (SURVEY.md §8(b)
// "sharded layer": sbbf_dist_create / insert / find / gather), in C++ for
// C/C++ callers; paper_2101_01719_b200/sharded.py is the same layer over
// torch.distributed for Python callers.
//
// One process (or thread) per GPU, one rank per GPU of an NCCL communicator
// the caller owns. Rank r owns global blocks [floor(rB/P), floor((r+1)B/P))
// (an sbbf_gpu shard that keeps the global block_index) and a receive window
// (sbbf_route.cu). Per collective call:
//   insert: dispatch (partition straight into the owners' windows over
//           NVLink) -> barrier -> insert_window
//   find:   dispatch -> barrier -> find_window -> barrier -> combine
// The barrier is a 1-element ncclAllReduce on the caller's stream, so the
// phases are stream-ordered with no host sync. Window handles (CUDA IPC)
// are exchanged once, at create, with an ncclAllGather.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing a copy the
// process already loaded, e.g. torch's), so the library itself loads — and
// the single-GPU ABI works — on machines without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "sbbf_internal.h"

namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclCommUserRank) comm_user_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclCommGetAsyncError) get_async_error = nullptr;
  decltype(&ncclCommAbort) comm_abort = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)?
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = "libnccl.so.2 not found";
      return;
    }
#define SBBF_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, #name))
    SBBF_SYM(get_unique_id, ncclGetUniqueId);
    SBBF_SYM(comm_init_rank, ncclCommInitRank);
    SBBF_SYM(comm_destroy, ncclCommDestroy);
    SBBF_SYM(comm_count, ncclCommCount);
    SBBF_SYM(comm_user_rank, ncclCommUserRank);
    SBBF_SYM(all_gather, ncclAllGather);
    SBBF_SYM(all_reduce, ncclAllReduce);
    SBBF_SYM(send, ncclSend);
    SBBF_SYM(recv, ncclRecv);
    SBBF_SYM(group_start, ncclGroupStart);
    SBBF_SYM(group_end, ncclGroupEnd);
    SBBF_SYM(error_string, ncclGetErrorString);
    SBBF_SYM(get_async_error, ncclCommGetAsyncError);
    SBBF_SYM(comm_abort, ncclCommAbort);
#undef SBBF_SYM
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.comm_count && n.comm_user_rank &&
           n.all_gather && n.all_reduce && n.send && n.recv && n.group_start && n.group_end && n.error_string &&
           n.get_async_error && n.comm_abort;
    if (!n.ok) n.why = "libnccl.so.2 lacks an expected symbol";
  });
  return n;
}

int dist_fail(int code, const std::string& msg) {
  sbbf::set_last_error(msg);
  return code;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SBBF_OK;
  return dist_fail(SBBF_ECUDA, std::string(what) + ": " + nccl().error_string(r));
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SBBF_OK;
  cudaGetLastError();
  return dist_fail(e == cudaErrorMemoryAllocation ? SBBF_ENOMEM : SBBF_ECUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

struct sbbf_dist {
  ncclComm_t comm = nullptr;      // NCCL mode (null in hooks mode)
  sbbf_dist_hooks hooks{};        // hooks mode: the caller's collectives
  bool use_hooks = false;
  bool aborted = false;           // a watchdog aborted the communicator: every call fails
  int rank = 0, world = 1, device = 0;
  uint64_t total = 0;
  std::vector<uint64_t> bounds;   // world + 1 entries
  uint64_t* d_bounds = nullptr;   // world entries (partition input)
  sbbf_gpu_t* shard = nullptr;
  sbbf_route_t* route = nullptr;
  int* d_flag = nullptr;          // barrier all-reduce buffer
};

namespace {

int barrier(sbbf_dist* d, cudaStream_t s) {
  if (d->aborted) return dist_fail(SBBF_ECUDA, "sharded filter: communicator aborted");
  if (d->world == 1) return SBBF_OK;
  if (d->use_hooks) {
    const int rc = d->hooks.barrier(d->hooks.ctx, s);
    return rc == 0 ? SBBF_OK : dist_fail(SBBF_ECUDA, "sharded filter: barrier hook failed");
  }
  return nccl_check(nccl().all_reduce(d->d_flag, d->d_flag, 1, ncclInt32, ncclSum, d->comm, s), "barrier");
}

// Host-side wait for `s` with NCCL failure detection: poll the stream and
// ncclCommGetAsyncError; on an asynchronous NCCL error (a peer died, a
// network fault) or after timeout_ms, abort the communicator
// (ncclCommAbort: the stuck kernels are torn down instead of spinning on a
// peer forever) and fail. timeout_ms <= 0 waits without a deadline.
int wait_stream(sbbf_dist* d, cudaStream_t s, long long timeout_ms, const char* what) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return SBBF_OK;
    if (q != cudaErrorNotReady) return cuda_check(q, what);
    if (!d->use_hooks && d->comm && d->world > 1) {
      ncclResult_t ae = ncclSuccess;
      nccl().get_async_error(d->comm, &ae);
      if (ae != ncclSuccess && ae != ncclInProgress) {
        nccl().comm_abort(d->comm);
        d->comm = nullptr;
        d->aborted = true;
        return dist_fail(SBBF_ECUDA, std::string(what) + ": NCCL asynchronous error (" + nccl().error_string(ae) +
                                         "); communicator aborted");
      }
    }
    const long long ms =
        std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && ms > timeout_ms) {
      if (!d->use_hooks && d->comm) {
        nccl().comm_abort(d->comm);
        d->comm = nullptr;
      }
      d->aborted = true;
      return dist_fail(SBBF_ECUDA, std::string(what) + ": timed out after " + std::to_string(ms) +
                                       " ms (a peer rank is not progressing); communicator aborted");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int sbbf_dist_unique_id(void* id) {
  if (!id) return dist_fail(SBBF_EINVAL, "sbbf_dist_unique_id: null buffer");
  if (!nccl().ok) return dist_fail(SBBF_ENODEV, "NCCL unavailable: " + nccl().why);
  ncclUniqueId u;
  const int rc = nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  if (rc == SBBF_OK) std::memcpy(id, &u, sizeof(u));
  return rc;
}

int sbbf_dist_comm_init(const void* id, int world, int rank, int device, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world)
    return dist_fail(SBBF_EINVAL, "sbbf_dist_comm_init: bad argument");
  if (!nccl().ok) return dist_fail(SBBF_ENODEV, "NCCL unavailable: " + nccl().why);
  Guard g(device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  const int rc = nccl_check(nccl().comm_init_rank(&c, world, u, rank), "ncclCommInitRank");
  *comm = rc == SBBF_OK ? c : nullptr;
  return rc;
}

int sbbf_dist_comm_destroy(void* comm) {
  if (!comm) return SBBF_OK;
  if (!nccl().ok) return dist_fail(SBBF_ENODEV, "NCCL unavailable: " + nccl().why);
  return nccl_check(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

int sbbf_dist_destroy(sbbf_dist_t* d) {
  if (!d) return SBBF_OK;
  Guard g(d->device);
  cudaDeviceSynchronize();
  sbbf_route_destroy(d->route);
  sbbf_gpu_destroy(d->shard);
  cudaFree(d->d_bounds);
  cudaFree(d->d_flag);
  cudaGetLastError();
  delete d;
  return SBBF_OK;
}

namespace {

// SBBF_DIST_DEBUG=1 traces the collective steps on stderr (hang diagnosis).
void trace(const sbbf_dist* d, const char* what) {
  static const bool on = getenv("SBBF_DIST_DEBUG") != nullptr;
  if (on) fprintf(stderr, "sbbf_dist rank %d/%d: %s\n", d->rank, d->world, what);
}

// Rank-order gather of `bytes` host bytes from every rank: ncclAllGather
// through a device buffer, or the caller's hook.
int allgather_host(sbbf_dist* d, const void* send, void* recv, uint64_t bytes) {
  if (d->world == 1) {
    std::memcpy(recv, send, bytes);
    return SBBF_OK;
  }
  if (d->use_hooks)
    return d->hooks.allgather(d->hooks.ctx, send, recv, bytes) == 0 ? SBBF_OK
                                                                      : dist_fail(SBBF_ECUDA, "allgather hook failed");
  uint8_t* dv = nullptr;
  int rc = cuda_check(cudaMalloc(&dv, bytes * d->world), "allgather");
  if (rc == SBBF_OK) rc = cuda_check(cudaMemcpy(dv + bytes * d->rank, send, bytes, cudaMemcpyHostToDevice), "allgather");
  if (rc == SBBF_OK)
    rc = nccl_check(nccl().all_gather(dv + bytes * d->rank, dv, bytes, ncclUint8, d->comm, nullptr), "ncclAllGather");
  if (rc == SBBF_OK) rc = wait_stream(d, nullptr, 600000, "allgather");
  if (rc == SBBF_OK) rc = cuda_check(cudaMemcpy(recv, dv, bytes * d->world, cudaMemcpyDeviceToHost), "allgather");
  cudaFree(dv);
  return rc;
}

// Shard, bounds, barrier flag and receive window; window handles exchanged
// with one rank-order gather; every rank maps every window before anyone
// dispatches.
int create_common(sbbf_dist* d, uint64_t total_buckets, uint64_t max_batch) {
  int rc = SBBF_OK;
  if (total_buckets < static_cast<uint64_t>(d->world))
    rc = dist_fail(SBBF_EINVAL, "sbbf_dist_create: fewer buckets than ranks");
  if (rc == SBBF_OK) {
    d->bounds.resize(d->world + 1);
    rc = sbbf_shard_bounds(total_buckets, static_cast<uint32_t>(d->world), d->bounds.data());
  }
  if (rc == SBBF_OK)
    rc = sbbf_gpu_create_shard(total_buckets, d->bounds[d->rank], d->bounds[d->rank + 1] - d->bounds[d->rank],
                               d->device, &d->shard);
  if (rc == SBBF_OK) rc = cuda_check(cudaMalloc(&d->d_bounds, d->world * sizeof(uint64_t)), "bounds");
  if (rc == SBBF_OK)
    rc = cuda_check(cudaMemcpy(d->d_bounds, d->bounds.data(), d->world * sizeof(uint64_t), cudaMemcpyHostToDevice),
                    "bounds");
  if (rc == SBBF_OK) rc = cuda_check(cudaMalloc(&d->d_flag, sizeof(int)), "barrier flag");
  if (rc == SBBF_OK) rc = cuda_check(cudaMemset(d->d_flag, 0, sizeof(int)), "barrier flag");
  if (rc == SBBF_OK)
    rc = sbbf_route_create(static_cast<uint32_t>(d->world), static_cast<uint32_t>(d->rank), max_batch, d->device,
                           &d->route);
  trace(d, rc == SBBF_OK ? "create: shard and window ready" : "create: shard/window failed");
  if (rc == SBBF_OK && d->world > 1) {
    std::vector<uint8_t> mine(64), all(static_cast<size_t>(64) * d->world);
    rc = sbbf_route_ipc_handle(d->route, mine.data());
    if (rc == SBBF_OK) rc = allgather_host(d, mine.data(), all.data(), 64);
    trace(d, "create: handles exchanged");
    for (int p = 0; rc == SBBF_OK && p < d->world; ++p)
      if (p != d->rank) rc = sbbf_route_open_peer(d->route, static_cast<uint32_t>(p), all.data() + 64 * p);
    trace(d, "create: peers mapped");
    if (rc == SBBF_OK) rc = barrier(d, nullptr);
    if (rc == SBBF_OK) rc = wait_stream(d, nullptr, 600000, "create");
    trace(d, "create: done");
  }
  return rc;
}

}  // namespace

int sbbf_dist_create(void* comm, uint64_t total_buckets, uint64_t max_batch, int device, sbbf_dist_t** out) {
  if (!comm || !out || total_buckets == 0 || max_batch == 0)
    return dist_fail(SBBF_EINVAL, "sbbf_dist_create: bad argument");
  *out = nullptr;
  if (!nccl().ok) return dist_fail(SBBF_ENODEV, "NCCL unavailable: " + nccl().why);
  Guard g(device);
  auto* d = new sbbf_dist;
  d->comm = static_cast<ncclComm_t>(comm);
  d->device = device;
  d->total = total_buckets;
  int rc = nccl_check(nccl().comm_count(d->comm, &d->world), "ncclCommCount");
  if (rc == SBBF_OK) rc = nccl_check(nccl().comm_user_rank(d->comm, &d->rank), "ncclCommUserRank");
  if (rc == SBBF_OK) rc = create_common(d, total_buckets, max_batch);
  if (rc != SBBF_OK) {
    d->comm = d->aborted ? nullptr : d->comm;
    sbbf_dist_destroy(d);
    return rc;
  }
  *out = d;
  return SBBF_OK;
}

int sbbf_dist_create_hooks(const sbbf_dist_hooks* hooks, uint64_t total_buckets, uint64_t max_batch, int device,
                           sbbf_dist_t** out) {
  if (!hooks || !out || total_buckets == 0 || max_batch == 0 || hooks->world < 1 || hooks->rank < 0 ||
      hooks->rank >= hooks->world || !hooks->allgather || !hooks->barrier)
    return dist_fail(SBBF_EINVAL, "sbbf_dist_create_hooks: bad argument");
  *out = nullptr;
  Guard g(device);
  auto* d = new sbbf_dist;
  d->hooks = *hooks;
  d->use_hooks = true;
  d->rank = hooks->rank;
  d->world = hooks->world;
  d->device = device;
  d->total = total_buckets;
  const int rc = create_common(d, total_buckets, max_batch);
  if (rc != SBBF_OK) {
    sbbf_dist_destroy(d);
    return rc;
  }
  *out = d;
  return SBBF_OK;
}

int sbbf_dist_sync(sbbf_dist_t* d, void* stream, int64_t timeout_ms) {
  if (!d) return dist_fail(SBBF_EINVAL, "sbbf_dist_sync: null handle");
  if (d->aborted) return dist_fail(SBBF_ECUDA, "sharded filter: communicator aborted");
  Guard g(d->device);
  return wait_stream(d, static_cast<cudaStream_t>(stream), timeout_ms, "sbbf_dist_sync");
}

int sbbf_dist_image_crc(sbbf_dist_t* d, uint32_t* crc) {
  if (!d || !crc) return dist_fail(SBBF_EINVAL, "sbbf_dist_image_crc: bad argument");
  if (d->aborted) return dist_fail(SBBF_ECUDA, "sharded filter: communicator aborted");
  Guard g(d->device);
  uint32_t mine = 0;
  int rc = sbbf_gpu_blocks_crc(d->shard, &mine);
  std::vector<uint32_t> all(d->world);
  if (rc == SBBF_OK) rc = allgather_host(d, &mine, all.data(), sizeof(uint32_t));
  if (rc != SBBF_OK) return rc;
  uint8_t hdr[17] = {'S', 'B', 'B', 'F', 1, 0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) hdr[9 + i] = static_cast<uint8_t>(d->total >> (8 * i));
  uint32_t c = sbbf_crc32_update(0, hdr, sizeof(hdr));
  for (int p = 0; p < d->world; ++p) c = sbbf_crc32_combine(c, all[p], (d->bounds[p + 1] - d->bounds[p]) * 32);
  *crc = c;
  return SBBF_OK;
}

int sbbf_dist_rank(const sbbf_dist_t* d) { return d ? d->rank : -1; }
int sbbf_dist_world(const sbbf_dist_t* d) { return d ? d->world : 0; }
sbbf_gpu_t* sbbf_dist_shard(sbbf_dist_t* d) { return d ? d->shard : nullptr; }

int sbbf_dist_insert(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, void* stream) {
  if (!d) return dist_fail(SBBF_EINVAL, "sbbf_dist_insert: null handle");
  Guard g(d->device);
  const auto s = static_cast<cudaStream_t>(stream);
  int rc = sbbf_route_dispatch(d->route, d_hashes, n, d->total, d->d_bounds, 0, stream);
  trace(d, "insert: dispatched");
  if (rc == SBBF_OK) rc = barrier(d, s);
  trace(d, "insert: barrier passed");
  if (rc == SBBF_OK) rc = sbbf_route_insert_window(d->route, d->shard, stream);
  trace(d, "insert: window inserted");
  return rc;
}

int sbbf_dist_find(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, uint8_t* d_results, void* stream) {
  if (!d) return dist_fail(SBBF_EINVAL, "sbbf_dist_find: null handle");
  Guard g(d->device);
  const auto s = static_cast<cudaStream_t>(stream);
  int rc = sbbf_route_dispatch(d->route, d_hashes, n, d->total, d->d_bounds, 1, stream);
  trace(d, "find: dispatched");
  if (rc == SBBF_OK) rc = barrier(d, s);
  trace(d, "find: barrier 1 passed");
  if (rc == SBBF_OK) rc = sbbf_route_find_window(d->route, d->shard, stream);
  trace(d, "find: window probed");
  if (rc == SBBF_OK) rc = barrier(d, s);
  trace(d, "find: barrier 2 passed");
  if (rc == SBBF_OK) rc = sbbf_route_combine(d->route, d_results, stream);
  trace(d, "find: combined");
  return rc;
}

int sbbf_dist_find_bits(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, uint32_t* d_bits, void* stream) {
  if (!d || (n && !d_bits)) return dist_fail(SBBF_EINVAL, "sbbf_dist_find_bits: bad argument");
  if (n == 0) return sbbf_dist_find(d, d_hashes, 0, nullptr, stream);
  Guard g(d->device);
  const auto s = static_cast<cudaStream_t>(stream);
  uint8_t* bytes = nullptr;
  int rc = cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&bytes), n, s), "find_bits");
  if (rc == SBBF_OK) rc = sbbf_dist_find(d, d_hashes, n, bytes, stream);
  if (rc == SBBF_OK) rc = sbbf_pack_bits(bytes, n, d_bits, stream);
  if (bytes) cudaFreeAsync(bytes, s);
  return rc;
}

// The whole filter on rank `root` (h_dst: total_buckets * 32 bytes there,
// ignored elsewhere): the shards in rank order, byte-identical to one
// total_buckets filter. Collective; synchronous.
int sbbf_dist_gather(sbbf_dist_t* d, void* h_dst, int root) {
  if (!d || root < 0 || root >= d->world || (d->rank == root && !h_dst))
    return dist_fail(SBBF_EINVAL, "sbbf_dist_gather: bad argument");
  if (d->aborted) return dist_fail(SBBF_ECUDA, "sharded filter: communicator aborted");
  Guard g(d->device);
  int rc = cuda_check(cudaDeviceSynchronize(), "gather");
  if (rc != SBBF_OK) return rc;
  const uint64_t mine = d->bounds[d->rank + 1] - d->bounds[d->rank];
  if (d->use_hooks || d->world == 1) {
    // every shard padded to the largest, gathered on the host in rank order
    uint64_t most = 0;
    for (int p = 0; p < d->world; ++p) most = std::max<uint64_t>(most, d->bounds[p + 1] - d->bounds[p]);
    std::vector<uint8_t> send(most * 32), all(most * 32 * d->world);
    rc = sbbf_gpu_to_host(d->shard, send.data(), mine * 32);
    if (rc == SBBF_OK) rc = allgather_host(d, send.data(), all.data(), most * 32);
    if (rc == SBBF_OK && d->rank == root)
      for (int p = 0; p < d->world; ++p)
        std::memcpy(static_cast<uint8_t*>(h_dst) + d->bounds[p] * 32, all.data() + most * 32 * p,
                    (d->bounds[p + 1] - d->bounds[p]) * 32);
    return rc;
  }
  if (d->rank != root) {
    rc = nccl_check(nccl().send(sbbf_gpu_device_blocks(d->shard), mine * 32, ncclUint8, root, d->comm, nullptr),
                    "ncclSend(shard)");
    if (rc == SBBF_OK) rc = wait_stream(d, nullptr, 600000, "gather");
    return rc;
  }
  auto* out = static_cast<uint8_t*>(h_dst);
  rc = sbbf_gpu_to_host(d->shard, out + d->bounds[d->rank] * 32, mine * 32);
  for (int p = 0; rc == SBBF_OK && p < d->world; ++p) {
    if (p == root) continue;
    const uint64_t cnt = d->bounds[p + 1] - d->bounds[p];
    uint8_t* stage = nullptr;
    rc = cuda_check(cudaMalloc(&stage, cnt * 32), "gather stage");
    if (rc == SBBF_OK) rc = nccl_check(nccl().recv(stage, cnt * 32, ncclUint8, p, d->comm, nullptr), "ncclRecv(shard)");
    if (rc == SBBF_OK) rc = wait_stream(d, nullptr, 600000, "gather");
    if (rc == SBBF_OK)
      rc = cuda_check(cudaMemcpy(out + d->bounds[p] * 32, stage, cnt * 32, cudaMemcpyDeviceToHost), "gather");
    cudaFree(stage);
  }
  return rc;
}

}  // extern "C"
