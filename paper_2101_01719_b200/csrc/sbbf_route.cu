// sbbf_route.cu — fused multi-GPU dispatch over peer memory (SURVEY.md §8(e),
// "fused option"; the reference itself has no distributed mode).
//
// The NCCL path (sharded.py) partitions a batch into a local staging array,
// exchanges counts (a host sync), then all-to-alls the keys. Here the
// partition's scatter writes every owner's run STRAIGHT INTO THAT OWNER'S
// RECEIVE WINDOW — a buffer on the owner GPU mapped into this process with
// CUDA IPC, written over NVLink/NVSwitch by ordinary coalesced stores — and
// publishes the run length next to it. No staging copy, no host round trip:
//
//   insert:  dispatch (count -> scan -> routed scatter)   [source]
//            collective barrier (stream-ordered)
//            insert_window: every key in my window         [owner]
//   lookup:  dispatch (+ source positions kept locally)    [source]
//            barrier
//            find_window: one answer byte per window slot  [owner]
//            barrier
//            combine: read my answers back from each owner's window over
//            NVLink (coalesced) and scatter them to source order [source]
//
// Window layout (one cudaMalloc per rank, exported by IPC handle), P parts,
// R = max keys per source per call, two parities so call k+1 can be
// dispatched while nobody still reads call k's buffers:
//   [0, 1 KiB)           counts[2][64]       u64, counts[p][src]
//   keys  (p, src)       at 1 KiB + ((p*P + src) * R) * 8
//   answers (p, src)     at 1 KiB + 2*P*R*8 + (p*P + src) * R
// Source `src` owns region (p, src) of every window, so regions never
// overlap and no atomics are needed. Parity flips at every dispatch; every
// rank dispatches exactly once per collective call, so parities agree.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "sbbf_device.cuh"
#include "sbbf_internal.h"

namespace sbbf {
namespace {

constexpr uint32_t kMaxParts = 64;
constexpr uint64_t kHeader = 1024;
constexpr int kWinThreads = 256;

__device__ __forceinline__ uint32_t region_of(const unsigned long long* prefix, uint32_t P, uint64_t i) {
  // largest r with prefix[r] <= i (prefix[0] = 0, prefix[P] = total > i)
  uint32_t lo = 0, hi = P;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void load_prefix(const unsigned long long* counts, uint32_t P,
                                            unsigned long long* prefix) {
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    prefix[0] = 0;
    for (uint32_t r = 0; r < P; ++r) {
      s += counts[r];
      prefix[r + 1] = s;
    }
  }
  __syncthreads();
}

// Owner: OR every key of this rank's window into the local shard. 4 threads
// per key, one red.global.or.b64 per lane pair (as insert_wide_kernel).
__global__ void __launch_bounds__(kWinThreads, 4) window_insert_kernel(uint32_t* __restrict__ blocks, Geom g,
                                                                       const unsigned long long* __restrict__ counts,
                                                                       const uint64_t* __restrict__ keys,
                                                                       uint64_t R, uint32_t P) {
  __shared__ unsigned long long prefix[kMaxParts + 1];
  load_prefix(counts, P, prefix);
  const uint64_t n = prefix[P];
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 2, pair = lane & 3;
  const uint32_t seed_lo = dev::lane_seed_rt(2 * pair), seed_hi = dev::lane_seed_rt(2 * pair + 1);
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t keep = dev::policy_evict_last();
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kWinThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kWinThreads) >> 5;
  const uint64_t ntiles = (n + 31) >> 5;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t idx = (t << 5) + lane;
    uint64_t h = 0;
    if (idx < n) {
      const uint32_t r = region_of(prefix, P, idx);
      SBBF_DCHECK(r < P && idx - prefix[r] < R);
      h = dev::ld_stream_u64(keys + r * R + (idx - prefix[r]), pol);
    }
    const uint32_t valid = __ballot_sync(0xffffffffu, idx < n);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = q * 8 + sub;
      const uint64_t hk = __shfl_sync(0xffffffffu, h, k);
      const uint64_t b = dev::block_index(hk, g.nb_global) - g.first;
      const bool ok = ((valid >> k) & 1u) && b < g.nb_local;
      if (ok) {
        const uint32_t low = static_cast<uint32_t>(hk);
        const uint64_t mask =
            (static_cast<uint64_t>(dev::lane_bit(low, seed_hi)) << 32) | dev::lane_bit(low, seed_lo);
        dev::red_or64(reinterpret_cast<uint64_t*>(blocks + b * 8) + pair, mask, keep);
      }
    }
  }
}

// Owner: one answer byte per window slot, written in place next to the key.
__global__ void __launch_bounds__(kWinThreads, 3) window_find_kernel(const uint32_t* __restrict__ blocks, Geom g,
                                                                     const unsigned long long* __restrict__ counts,
                                                                     const uint64_t* __restrict__ keys,
                                                                     uint8_t* __restrict__ answers, uint64_t R,
                                                                     uint32_t P) {
  __shared__ unsigned long long prefix[kMaxParts + 1];
  load_prefix(counts, P, prefix);
  const uint64_t n = prefix[P];
  constexpr int U = 4;
  const uint64_t pol = dev::policy_evict_first();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWinThreads * U;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kWinThreads * U + threadIdx.x; base < n;
       base += stride) {
    uint64_t h[U], slot[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = base + static_cast<uint64_t>(u) * kWinThreads;
      slot[u] = ~0ull;
      h[u] = 0;
      if (idx < n) {
        const uint32_t r = region_of(prefix, P, idx);
        SBBF_DCHECK(r < P && idx - prefix[r] < R);
        slot[u] = r * R + (idx - prefix[r]);
        h[u] = dev::ld_stream_u64(keys + slot[u], pol);
      }
    }
    dev::Block8 b[U];
    uint32_t owned = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t blk = dev::block_index(h[u], g.nb_global) - g.first;
      const bool ok = blk < g.nb_local;
      owned |= static_cast<uint32_t>(ok) << u;
      dev::ld_block_nc(blocks + (ok ? blk : 0) * 8, b[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (slot[u] != ~0ull)
        answers[slot[u]] = (((owned >> u) & 1u) && dev::block_contains(b[u], h[u])) ? 1 : 0;
  }
}

// Source: answers back from every owner's window (coalesced NVLink reads of
// this source's region) to source order.
__global__ void __launch_bounds__(kWinThreads) combine_kernel(const unsigned long long* __restrict__ counts,
                                                              const uint8_t* const* __restrict__ res_src,
                                                              uint32_t P, const uint32_t* __restrict__ pos,
                                                              uint64_t n, uint8_t* __restrict__ out) {
  __shared__ unsigned long long prefix[kMaxParts + 1];
  __shared__ const uint8_t* src[kMaxParts];
  if (threadIdx.x < P) src[threadIdx.x] = res_src[threadIdx.x];
  load_prefix(counts, P, prefix);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWinThreads;
  for (uint64_t s = static_cast<uint64_t>(blockIdx.x) * kWinThreads + threadIdx.x; s < n; s += stride) {
    const uint32_t r = region_of(prefix, P, s);
    SBBF_DCHECK(r < P && pos[s] < n);
    out[pos[s]] = src[r][s - prefix[r]];
  }
}

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace
}  // namespace sbbf

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct sbbf_route {
  uint32_t parts = 0, rank = 0;
  int device = 0;
  sbbf::DeviceInfo di;
  uint64_t R = 0;                 // max keys per source per call (region capacity)
  uint8_t* window = nullptr;      // this rank's receive window (IPC-exported)
  uint64_t window_bytes = 0;
  std::vector<uint8_t*> peer;     // peer window bases (peer[rank] = window)
  std::vector<bool> opened;       // peer mapped via cudaIpcOpenMemHandle (close on destroy)
  // device tables per parity: dst[p][b], count_dst[p][b], res_src[p][b]
  void** d_tables = nullptr;
  uint64_t* d_counts = nullptr;   // this source's per-destination counts (last dispatch)
  uint32_t* d_pos = nullptr;      // source index of every routed slot (last lookup dispatch)
  uint64_t last_n = 0;
  int parity = 1;                 // flipped at every dispatch: the first call uses parity 0
  bool positions = false;
};

namespace {

int route_fail(int code, const std::string& msg) {
  sbbf::set_last_error(msg);
  return code;
}

int route_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SBBF_OK;
  cudaGetLastError();
  return route_fail(e == cudaErrorMemoryAllocation ? SBBF_ENOMEM : SBBF_ECUDA,
                    std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t keys_off(const sbbf_route* rt, int p, uint32_t src) {
  return sbbf::kHeader + ((static_cast<uint64_t>(p) * rt->parts + src) * rt->R) * 8;
}
uint64_t res_off(const sbbf_route* rt, int p, uint32_t src) {
  return sbbf::kHeader + 2ull * rt->parts * rt->R * 8 + (static_cast<uint64_t>(p) * rt->parts + src) * rt->R;
}
uint64_t count_off(int p, uint32_t src) { return (static_cast<uint64_t>(p) * sbbf::kMaxParts + src) * 8; }

bool all_linked(const sbbf_route* rt) {
  for (auto* p : rt->peer)
    if (!p) return false;
  return true;
}

// Device tables: [p][3][64] pointers (dst keys, count slot, answer region).
int upload_tables(sbbf_route* rt) {
  if (!all_linked(rt)) return SBBF_OK;  // uploaded once the last peer is linked
  std::vector<void*> t(2 * 3 * sbbf::kMaxParts, nullptr);
  for (int p = 0; p < 2; ++p)
    for (uint32_t b = 0; b < rt->parts; ++b) {
      t[(p * 3 + 0) * sbbf::kMaxParts + b] = rt->peer[b] + keys_off(rt, p, rt->rank);
      t[(p * 3 + 1) * sbbf::kMaxParts + b] = rt->peer[b] + count_off(p, rt->rank);
      t[(p * 3 + 2) * sbbf::kMaxParts + b] = rt->peer[b] + res_off(rt, p, rt->rank);
    }
  return route_cuda(cudaMemcpy(rt->d_tables, t.data(), t.size() * sizeof(void*), cudaMemcpyHostToDevice),
                    "route tables");
}

void** table(const sbbf_route* rt, int p, int kind) {
  return rt->d_tables + (p * 3 + kind) * sbbf::kMaxParts;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

uint64_t sbbf_route_window_bytes(uint32_t parts, uint64_t max_batch) {
  const uint64_t R = sbbf::round_up(max_batch ? max_batch : 1, 256);
  return sbbf::kHeader + 2ull * parts * R * 9;
}

int sbbf_route_create(uint32_t parts, uint32_t rank, uint64_t max_batch, int device, sbbf_route_t** out) {
  if (!out || parts == 0 || parts > sbbf::kMaxParts || rank >= parts || max_batch == 0 ||
      max_batch > 0xffffffffull)
    return route_fail(SBBF_EINVAL, "sbbf_route_create: need 1 <= parts <= 64, rank < parts, "
                                   "0 < max_batch < 2^32");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return route_fail(SBBF_ENODEV, "sbbf_route_create: no CUDA device (there is no CPU fallback)");
  }
  DeviceGuard g(device);
  auto* rt = new sbbf_route;
  rt->parts = parts;
  rt->rank = rank;
  rt->device = device;
  rt->di.device = device;
  cudaDeviceGetAttribute(&rt->di.sms, cudaDevAttrMultiProcessorCount, device);
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device) == cudaSuccess && l2 > 0)
    rt->di.l2_bytes = static_cast<size_t>(l2);
  rt->R = sbbf::round_up(max_batch, 256);
  rt->window_bytes = sbbf_route_window_bytes(parts, max_batch);
  rt->peer.assign(parts, nullptr);
  rt->opened.assign(parts, false);
  int rc = route_cuda(cudaMalloc(&rt->window, rt->window_bytes), "route window");
  if (rc == SBBF_OK) rc = route_cuda(cudaMemset(rt->window, 0, sbbf::kHeader), "route window");
  if (rc == SBBF_OK)
    rc = route_cuda(cudaMalloc(reinterpret_cast<void**>(&rt->d_tables), 2 * 3 * sbbf::kMaxParts * sizeof(void*)),
                    "route tables");
  if (rc == SBBF_OK) rc = route_cuda(cudaMalloc(reinterpret_cast<void**>(&rt->d_counts), sbbf::kMaxParts * 8), "route counts");
  if (rc == SBBF_OK) rc = route_cuda(cudaMalloc(reinterpret_cast<void**>(&rt->d_pos), rt->R * 4), "route positions");
  if (rc != SBBF_OK) {
    sbbf_route_destroy(rt);
    return rc;
  }
  rt->peer[rank] = rt->window;
  rc = upload_tables(rt);
  if (rc != SBBF_OK) {
    sbbf_route_destroy(rt);
    return rc;
  }
  *out = rt;
  return SBBF_OK;
}

void sbbf_route_destroy(sbbf_route_t* rt) {
  if (!rt) return;
  DeviceGuard g(rt->device);
  cudaDeviceSynchronize();
  for (uint32_t b = 0; b < rt->parts; ++b)
    if (rt->opened[b] && rt->peer[b]) cudaIpcCloseMemHandle(rt->peer[b]);
  cudaFree(rt->window);
  cudaFree(rt->d_tables);
  cudaFree(rt->d_counts);
  cudaFree(rt->d_pos);
  cudaGetLastError();
  delete rt;
}

uint64_t sbbf_route_max_batch(const sbbf_route_t* rt) { return rt ? rt->R : 0; }

int sbbf_route_ipc_handle(const sbbf_route_t* rt, void* handle) {
  if (!rt || !handle) return route_fail(SBBF_EINVAL, "sbbf_route_ipc_handle: null argument");
  DeviceGuard g(rt->device);
  cudaIpcMemHandle_t h;
  const int rc = route_cuda(cudaIpcGetMemHandle(&h, rt->window), "cudaIpcGetMemHandle");
  if (rc == SBBF_OK) std::memcpy(handle, &h, sizeof(h));
  return rc;
}

int sbbf_route_open_peer(sbbf_route_t* rt, uint32_t peer, const void* handle) {
  if (!rt || !handle || peer >= rt->parts || peer == rt->rank)
    return route_fail(SBBF_EINVAL, "sbbf_route_open_peer: bad peer");
  if (rt->peer[peer]) return route_fail(SBBF_EINVAL, "sbbf_route_open_peer: peer already linked");
  DeviceGuard g(rt->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  const int rc = route_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  if (rc != SBBF_OK) return rc;
  rt->peer[peer] = static_cast<uint8_t*>(p);
  rt->opened[peer] = true;
  return upload_tables(rt);
}

int sbbf_route_link_local(sbbf_route_t* rt, uint32_t peer, const sbbf_route_t* other) {
  if (!rt || !other || peer >= rt->parts || other->parts != rt->parts || other->R != rt->R ||
      other->rank != peer)
    return route_fail(SBBF_EINVAL, "sbbf_route_link_local: contexts do not match (parts, max_batch, rank)");
  if (peer == rt->rank) return SBBF_OK;
  if (other->device != rt->device) {
    DeviceGuard g(rt->device);
    int can = 0;
    cudaDeviceCanAccessPeer(&can, rt->device, other->device);
    if (!can) return route_fail(SBBF_ENODEV, "sbbf_route_link_local: no peer access between the devices");
    const cudaError_t e = cudaDeviceEnablePeerAccess(other->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return route_cuda(e, "peer access");
    cudaGetLastError();
  }
  rt->peer[peer] = other->window;
  rt->opened[peer] = false;
  return upload_tables(rt);
}

int sbbf_route_ready(const sbbf_route_t* rt) { return rt && all_linked(rt) ? 1 : 0; }

int sbbf_route_dispatch(sbbf_route_t* rt, const uint64_t* d_hashes, uint64_t n, uint64_t total_buckets,
                        const uint64_t* d_bounds, int keep_positions, void* stream) {
  if (!rt || !d_bounds || (n && !d_hashes) || total_buckets < rt->parts)
    return route_fail(SBBF_EINVAL, "sbbf_route_dispatch: bad argument");
  if (n > rt->R) return route_fail(SBBF_EINVAL, "sbbf_route_dispatch: batch exceeds max_batch");
  if (!all_linked(rt)) return route_fail(SBBF_EINVAL, "sbbf_route_dispatch: peer windows not linked");
  DeviceGuard g(rt->device);
  rt->parity ^= 1;
  rt->last_n = n;
  rt->positions = keep_positions != 0;
  const int p = rt->parity;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return route_cuda(sbbf::route_partition(rt->di, total_buckets, rt->parts, d_bounds, d_hashes, n, rt->d_counts,
                                          keep_positions ? rt->d_pos : nullptr,
                                          reinterpret_cast<uint64_t* const*>(table(rt, p, 0)),
                                          reinterpret_cast<unsigned long long* const*>(table(rt, p, 1)), s),
                    "sbbf_route_dispatch");
}

}  // extern "C"

namespace {
// Shards beyond 2 x L2 (config 5's 1 GiB shards at P = 8): random probes
// would be DRAM-bound, so each source region goes through the shard's own
// AUTO dispatch (the L2-blocked path) instead of the direct window kernel.
// That needs the region counts on the host: one small copy + stream sync.
bool window_blocked(const sbbf_route* rt, const sbbf_gpu_t* shard) {
  return sbbf_gpu_size_bytes(shard) > 2 * static_cast<uint64_t>(rt->di.l2_bytes);
}

int window_counts(const sbbf_route* rt, int p, cudaStream_t s, uint64_t* h) {
  int rc = route_cuda(cudaMemcpyAsync(h, rt->window + count_off(p, 0), rt->parts * sizeof(uint64_t),
                                      cudaMemcpyDeviceToHost, s),
                      "window counts");
  if (rc == SBBF_OK) rc = route_cuda(cudaStreamSynchronize(s), "window counts");
  return rc;
}

// The source regions of window parity p copied back to back into one
// stream-ordered allocation (*keys, *total keys).
int gather_regions(const sbbf_route* rt, int p, const std::vector<uint64_t>& cnt, cudaStream_t s, uint64_t** keys,
                   uint64_t* total) {
  uint64_t t = 0;
  for (uint64_t c : cnt) t += c;
  *total = t;
  *keys = nullptr;
  if (t == 0) return SBBF_OK;
  int rc = route_cuda(cudaMallocAsync(reinterpret_cast<void**>(keys), t * sizeof(uint64_t), s), "window gather");
  for (uint64_t r = 0, off = 0; rc == SBBF_OK && r < rt->parts; off += cnt[r], ++r)
    if (cnt[r])
      rc = route_cuda(cudaMemcpyAsync(*keys + off, rt->window + keys_off(rt, p, static_cast<uint32_t>(r)),
                                      cnt[r] * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s),
                      "window gather");
  return rc;
}
}  // namespace

extern "C" {

int sbbf_route_insert_window(sbbf_route_t* rt, sbbf_gpu_t* shard, void* stream) {
  if (!rt || !shard) return route_fail(SBBF_EINVAL, "sbbf_route_insert_window: null argument");
  DeviceGuard g(rt->device);
  const int p = rt->parity;
  if (window_blocked(rt, shard)) {
    std::vector<uint64_t> cnt(rt->parts);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = window_counts(rt, p, s, cnt.data());
    // the regions go straight into one blocked pass (one sweep of the shard
    // through L2, no staging copy) ...
    std::vector<const uint64_t*> ptrs(rt->parts);
    for (uint32_t r = 0; r < rt->parts; ++r)
      ptrs[r] = reinterpret_cast<const uint64_t*>(rt->window + keys_off(rt, p, r));
    bool handled = false;
    if (rc == SBBF_OK) rc = sbbf::gpu_insert_regions(shard, ptrs.data(), cnt.data(), rt->parts, s, &handled);
    if (rc != SBBF_OK || handled) return rc;
    // ... or, when the shard's plan cannot take regions, into one gathered batch
    uint64_t* keys = nullptr;
    uint64_t total = 0;
    if (rc == SBBF_OK) rc = gather_regions(rt, p, cnt, s, &keys, &total);
    if (rc == SBBF_OK && total) rc = sbbf_gpu_insert_batch(shard, keys, total, stream);
    if (keys) cudaFreeAsync(keys, s);
    return rc;
  }
  const sbbf::Geom geom{sbbf_gpu_total_buckets(shard), sbbf_gpu_first_block(shard), sbbf_gpu_num_buckets(shard)};
  sbbf::note_launch();
  // the window holds at most parts * R keys; the grid strides over the real count
  sbbf::window_insert_kernel<<<static_cast<unsigned>(rt->di.sms * 4), sbbf::kWinThreads, 0,
                               static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint32_t*>(sbbf_gpu_device_blocks(shard)), geom,
      reinterpret_cast<const unsigned long long*>(rt->window + count_off(p, 0)),
      reinterpret_cast<const uint64_t*>(rt->window + keys_off(rt, p, 0)), rt->R, rt->parts);
  return route_cuda(cudaGetLastError(), "window_insert_kernel");
}

int sbbf_route_find_window(sbbf_route_t* rt, const sbbf_gpu_t* shard, void* stream) {
  if (!rt || !shard) return route_fail(SBBF_EINVAL, "sbbf_route_find_window: null argument");
  DeviceGuard g(rt->device);
  const int p = rt->parity;
  if (window_blocked(rt, shard)) {
    std::vector<uint64_t> cnt(rt->parts);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = window_counts(rt, p, s, cnt.data());
    std::vector<const uint64_t*> ptrs(rt->parts);
    std::vector<uint8_t*> outs(rt->parts);
    for (uint32_t r = 0; r < rt->parts; ++r) {
      ptrs[r] = reinterpret_cast<const uint64_t*>(rt->window + keys_off(rt, p, r));
      outs[r] = rt->window + res_off(rt, p, r);
    }
    bool handled = false;
    if (rc == SBBF_OK) rc = sbbf::gpu_find_regions(shard, ptrs.data(), cnt.data(), rt->parts, outs.data(), s, &handled);
    if (rc != SBBF_OK || handled) return rc;
    uint64_t* keys = nullptr;
    uint64_t total = 0;
    uint8_t* ans = nullptr;
    if (rc == SBBF_OK) rc = gather_regions(rt, p, cnt, s, &keys, &total);
    if (rc == SBBF_OK && total) rc = route_cuda(cudaMallocAsync(reinterpret_cast<void**>(&ans), total, s), "answers");
    if (rc == SBBF_OK && total) rc = sbbf_gpu_find_batch(shard, keys, total, ans, stream);
    // answers back next to each source region
    for (uint64_t r = 0, off = 0; rc == SBBF_OK && r < rt->parts; off += cnt[r], ++r)
      if (cnt[r])
        rc = route_cuda(cudaMemcpyAsync(rt->window + res_off(rt, p, static_cast<uint32_t>(r)), ans + off, cnt[r],
                                        cudaMemcpyDeviceToDevice, s),
                        "answers");
    if (keys) cudaFreeAsync(keys, s);
    if (ans) cudaFreeAsync(ans, s);
    return rc;
  }
  const sbbf::Geom geom{sbbf_gpu_total_buckets(shard), sbbf_gpu_first_block(shard), sbbf_gpu_num_buckets(shard)};
  sbbf::note_launch();
  sbbf::window_find_kernel<<<static_cast<unsigned>(rt->di.sms * 3), sbbf::kWinThreads, 0,
                             static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint32_t*>(sbbf_gpu_device_blocks(const_cast<sbbf_gpu_t*>(shard))), geom,
      reinterpret_cast<const unsigned long long*>(rt->window + count_off(p, 0)),
      reinterpret_cast<const uint64_t*>(rt->window + keys_off(rt, p, 0)), rt->window + res_off(rt, p, 0), rt->R,
      rt->parts);
  return route_cuda(cudaGetLastError(), "window_find_kernel");
}

int sbbf_route_combine(sbbf_route_t* rt, uint8_t* d_results, void* stream) {
  if (!rt || (rt->last_n && !d_results)) return route_fail(SBBF_EINVAL, "sbbf_route_combine: null argument");
  if (!rt->positions) return route_fail(SBBF_EINVAL, "sbbf_route_combine: last dispatch kept no positions");
  if (rt->last_n == 0) return SBBF_OK;
  DeviceGuard g(rt->device);
  sbbf::note_launch();
  const uint64_t grid = sbbf::grid_for(rt->last_n, 2048, rt->di.sms, 8);
  sbbf::combine_kernel<<<static_cast<unsigned>(grid), sbbf::kWinThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(rt->d_counts),
      reinterpret_cast<const uint8_t* const*>(table(rt, rt->parity, 2)), rt->parts, rt->d_pos, rt->last_n,
      d_results);
  return route_cuda(cudaGetLastError(), "combine_kernel");
}

}  // extern "C"
