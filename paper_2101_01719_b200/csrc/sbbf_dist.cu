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

#include <cstdint>
#include <cstring>
#include <mutex>
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
#undef SBBF_SYM
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.comm_count && n.comm_user_rank &&
           n.all_gather && n.all_reduce && n.send && n.recv && n.group_start && n.group_end && n.error_string;
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
  ncclComm_t comm = nullptr;
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
  if (d->world == 1) return SBBF_OK;
  return nccl_check(nccl().all_reduce(d->d_flag, d->d_flag, 1, ncclInt32, ncclSum, d->comm, s), "barrier");
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
  if (rc == SBBF_OK && total_buckets < static_cast<uint64_t>(d->world))
    rc = dist_fail(SBBF_EINVAL, "sbbf_dist_create: fewer buckets than ranks");
  if (rc == SBBF_OK) {
    d->bounds.resize(d->world + 1);
    rc = sbbf_shard_bounds(total_buckets, static_cast<uint32_t>(d->world), d->bounds.data());
  }
  if (rc == SBBF_OK)
    rc = sbbf_gpu_create_shard(total_buckets, d->bounds[d->rank], d->bounds[d->rank + 1] - d->bounds[d->rank],
                               device, &d->shard);
  if (rc == SBBF_OK) rc = cuda_check(cudaMalloc(&d->d_bounds, d->world * sizeof(uint64_t)), "bounds");
  if (rc == SBBF_OK)
    rc = cuda_check(cudaMemcpy(d->d_bounds, d->bounds.data(), d->world * sizeof(uint64_t), cudaMemcpyHostToDevice),
                    "bounds");
  if (rc == SBBF_OK) rc = cuda_check(cudaMalloc(&d->d_flag, sizeof(int)), "barrier flag");
  if (rc == SBBF_OK) rc = cuda_check(cudaMemset(d->d_flag, 0, sizeof(int)), "barrier flag");
  if (rc == SBBF_OK)
    rc = sbbf_route_create(static_cast<uint32_t>(d->world), static_cast<uint32_t>(d->rank), max_batch, device,
                           &d->route);
  if (rc == SBBF_OK && d->world > 1) {
    // exchange the window handles (one ncclAllGather of 64-byte records)
    uint8_t* d_handles = nullptr;
    std::vector<uint8_t> h(static_cast<size_t>(64) * d->world);
    rc = sbbf_route_ipc_handle(d->route, h.data() + 64 * d->rank);
    if (rc == SBBF_OK) rc = cuda_check(cudaMalloc(&d_handles, h.size()), "handles");
    if (rc == SBBF_OK) rc = cuda_check(cudaMemcpy(d_handles + 64 * d->rank, h.data() + 64 * d->rank, 64,
                                                  cudaMemcpyHostToDevice), "handles");
    if (rc == SBBF_OK)
      rc = nccl_check(nccl().all_gather(d_handles + 64 * d->rank, d_handles, 64, ncclUint8, d->comm, nullptr),
                      "ncclAllGather(handles)");
    if (rc == SBBF_OK) rc = cuda_check(cudaMemcpy(h.data(), d_handles, h.size(), cudaMemcpyDeviceToHost), "handles");
    cudaFree(d_handles);
    for (int p = 0; rc == SBBF_OK && p < d->world; ++p)
      if (p != d->rank) rc = sbbf_route_open_peer(d->route, static_cast<uint32_t>(p), h.data() + 64 * p);
    // every rank has mapped every window before anyone dispatches
    if (rc == SBBF_OK) rc = barrier(d, nullptr);
    if (rc == SBBF_OK) rc = cuda_check(cudaDeviceSynchronize(), "create");
  }
  if (rc != SBBF_OK) {
    sbbf_dist_destroy(d);
    return rc;
  }
  *out = d;
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
  if (rc == SBBF_OK) rc = barrier(d, s);
  if (rc == SBBF_OK) rc = sbbf_route_insert_window(d->route, d->shard, stream);
  return rc;
}

int sbbf_dist_find(sbbf_dist_t* d, const uint64_t* d_hashes, uint64_t n, uint8_t* d_results, void* stream) {
  if (!d) return dist_fail(SBBF_EINVAL, "sbbf_dist_find: null handle");
  Guard g(d->device);
  const auto s = static_cast<cudaStream_t>(stream);
  int rc = sbbf_route_dispatch(d->route, d_hashes, n, d->total, d->d_bounds, 1, stream);
  if (rc == SBBF_OK) rc = barrier(d, s);
  if (rc == SBBF_OK) rc = sbbf_route_find_window(d->route, d->shard, stream);
  if (rc == SBBF_OK) rc = barrier(d, s);
  if (rc == SBBF_OK) rc = sbbf_route_combine(d->route, d_results, stream);
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
  Guard g(d->device);
  int rc = cuda_check(cudaDeviceSynchronize(), "gather");
  if (rc != SBBF_OK) return rc;
  const uint64_t mine = d->bounds[d->rank + 1] - d->bounds[d->rank];
  if (d->rank != root) {
    rc = nccl_check(nccl().send(sbbf_gpu_device_blocks(d->shard), mine * 32, ncclUint8, root, d->comm, nullptr),
                    "ncclSend(shard)");
    if (rc == SBBF_OK) rc = cuda_check(cudaDeviceSynchronize(), "gather");
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
    if (rc == SBBF_OK)
      rc = cuda_check(cudaMemcpy(out + d->bounds[p] * 32, stage, cnt * 32, cudaMemcpyDeviceToHost), "gather");
    cudaFree(stage);
  }
  return rc;
}

}  // extern "C"
