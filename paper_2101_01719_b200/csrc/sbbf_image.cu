// sbbf_image.cu — FilterImage v1 on device: CRC-32 (IEEE, reflected 0xEDB88320)
// of the block array computed on the GPU (persist.cpp:64-70 is the
// byte-serial reference), for sbbf_gpu_serialize / sbbf_gpu_deserialize /
// sbbf_gpu_image_crc (image layout: persist.hpp:14-30).
//
// Parallel CRC: CRC is linear over GF(2), so crc(A||B) =
// crc(A) * x^(8|B|) mod P  xor  crc(B) (the "combine" identity zlib's
// crc32_combine uses). Each CTA stages a 64 KiB segment into shared memory
// with a bulk async copy (cp.async.bulk + mbarrier), every thread CRCs a
// 256-byte piece with slicing-by-8 tables in smem, pieces are combined in a
// tree inside the CTA (x^(8*256*2^k) operators precomputed on the host), and
// the host combines the per-segment CRCs.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "sbbf_internal.h"

namespace sbbf {
namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int kCrcThreads = 256;
constexpr uint32_t kPiece = 256;                       // bytes per thread
constexpr uint32_t kSegment = kCrcThreads * kPiece;    // 64 KiB per CTA
constexpr int kLevels = 8;                             // log2(kCrcThreads)

// a(x) * b(x) mod P(x) in the reflected representation (x^0 at bit 31).
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^(8 * nbytes) mod P by square-and-multiply.
uint32_t xpow8n(uint64_t nbytes) {
  uint32_t sq = 1u << 30;  // x^1
  for (int i = 0; i < 3; ++i) sq = multmodp(sq, sq);  // x^8
  uint32_t p = 1u << 31;   // x^0
  while (nbytes) {
    if (nbytes & 1) p = multmodp(sq, p);
    sq = multmodp(sq, sq);
    nbytes >>= 1;
  }
  return p;
}

struct CrcOps {
  uint32_t level[kLevels];  // x^(8 * kPiece * 2^k) mod P
};

__global__ void __launch_bounds__(kCrcThreads) crc_segments_kernel(const uint8_t* __restrict__ data,
                                                                   uint64_t bytes, CrcOps ops,
                                                                   uint32_t* __restrict__ seg_crc) {
  extern __shared__ __align__(128) uint8_t seg[];  // kSegment bytes (dynamic: > 48 KiB)
  __shared__ uint32_t table[8][256];
  __shared__ uint32_t part[kCrcThreads];
  __shared__ __align__(8) uint64_t mbar;
  const uint32_t t = threadIdx.x;
  // slicing-by-8 tables (table[0] is the byte-serial table of persist.cpp:15-28)
  {
    uint32_t c = t;
    for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
    table[0][t] = c;
  }
  __syncthreads();
  for (int k = 1; k < 8; ++k) {
    const uint32_t prev = table[k - 1][t];
    table[k][t] = (prev >> 8) ^ table[0][prev & 0xFFu];
    __syncthreads();
  }
  const uint64_t off = static_cast<uint64_t>(blockIdx.x) * kSegment;
  const uint32_t len = static_cast<uint32_t>(bytes - off < kSegment ? bytes - off : kSegment);
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar));
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(len) : "memory");
    for (uint32_t o = 0; o < len; o += 16384) {
      const uint32_t sz = len - o < 16384 ? len - o : 16384;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<uint32_t>(__cvta_generic_to_shared(seg + o))),
          "l"(data + off + o), "r"(sz), "r"(bar)
          : "memory");
    }
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar)
          : "memory");
  }
  // standard CRC-32 of this thread's piece (pieces are whole: len is a
  // multiple of kPiece because the block array is 32 * nb bytes and the
  // host only launches full pieces; a short piece CRCs what it has).
  const uint32_t pb = t * kPiece;
  const uint32_t plen = pb >= len ? 0 : (len - pb < kPiece ? len - pb : kPiece);
  uint32_t c = 0xFFFFFFFFu;
  const uint8_t* q = seg + pb;
  uint32_t i = 0;
  for (; i + 8 <= plen; i += 8) {
    const uint32_t lo = (static_cast<uint32_t>(q[i]) | (static_cast<uint32_t>(q[i + 1]) << 8) |
                         (static_cast<uint32_t>(q[i + 2]) << 16) | (static_cast<uint32_t>(q[i + 3]) << 24)) ^ c;
    const uint32_t hi = static_cast<uint32_t>(q[i + 4]) | (static_cast<uint32_t>(q[i + 5]) << 8) |
                        (static_cast<uint32_t>(q[i + 6]) << 16) | (static_cast<uint32_t>(q[i + 7]) << 24);
    c = table[7][lo & 0xFF] ^ table[6][(lo >> 8) & 0xFF] ^ table[5][(lo >> 16) & 0xFF] ^ table[4][lo >> 24] ^
        table[3][hi & 0xFF] ^ table[2][(hi >> 8) & 0xFF] ^ table[1][(hi >> 16) & 0xFF] ^ table[0][hi >> 24];
  }
  for (; i < plen; ++i) c = (c >> 8) ^ table[0][(c ^ q[i]) & 0xFFu];
  part[t] = c ^ 0xFFFFFFFFu;
  __syncthreads();
  // tree combine: pieces [j, j+2^(k+1)) from left/right halves of 2^k pieces
  for (int k = 0; k < kLevels; ++k) {
    const uint32_t span = 1u << (k + 1);
    if ((t & (span - 1)) == 0) {
      const uint32_t right = t + (span >> 1);
      const uint32_t rb = right * kPiece;
      if (rb < len) {
        const uint32_t rlen = len - rb < (span >> 1) * kPiece ? len - rb : (span >> 1) * kPiece;
        // full right halves use the precomputed operator; the ragged tail
        // (last segment only) falls back to computing it
        uint32_t op = ops.level[k];
        if (rlen != (span >> 1) * kPiece) {
          uint32_t sq = 1u << 30;
          for (int s2 = 0; s2 < 3; ++s2) sq = multmodp(sq, sq);
          op = 1u << 31;
          for (uint32_t n = rlen; n; n >>= 1) {
            if (n & 1) op = multmodp(sq, op);
            sq = multmodp(sq, sq);
          }
        }
        part[t] = multmodp(op, part[t]) ^ part[right];
      }
    }
    __syncthreads();
  }
  if (t == 0) seg_crc[blockIdx.x] = part[0];
}

}  // namespace

uint32_t crc32_host_update(uint32_t crc, const uint8_t* p, uint64_t n) {
  // byte-serial standard CRC-32 continuation for the 17-byte header
  uint32_t c = crc ^ 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) {
    c ^= p[i];
    for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
  }
  return c ^ 0xFFFFFFFFu;
}

uint32_t crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
  return multmodp(xpow8n(len2), crc1) ^ crc2;
}

cudaError_t device_crc32(const void* d_data, uint64_t bytes, uint32_t* crc_out, cudaStream_t s) {
  if (bytes == 0) {
    *crc_out = 0;
    return cudaSuccess;
  }
  const uint64_t nseg = (bytes + kSegment - 1) / kSegment;
  CrcOps ops;
  for (int k = 0; k < kLevels; ++k) ops.level[k] = xpow8n(static_cast<uint64_t>(kPiece) << k);
  uint32_t* d_seg = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_seg), nseg * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  static const cudaError_t attr =
      cudaFuncSetAttribute(crc_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSegment);
  if (attr != cudaSuccess) return attr;
  note_launch();
  crc_segments_kernel<<<static_cast<unsigned>(nseg), kCrcThreads, kSegment, s>>>(
      static_cast<const uint8_t*>(d_data), bytes, ops, d_seg);
  e = cudaGetLastError();
  std::vector<uint32_t> seg(nseg);
  if (e == cudaSuccess) e = cudaMemcpyAsync(seg.data(), d_seg, nseg * sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d_seg, s);
  if (e != cudaSuccess) return e;
  const uint32_t op_full = xpow8n(kSegment);
  uint32_t crc = seg[0];
  for (uint64_t i = 1; i < nseg; ++i) {
    const uint64_t len = (i == nseg - 1) ? bytes - i * kSegment : kSegment;
    crc = multmodp(len == kSegment ? op_full : xpow8n(len), crc) ^ seg[i];
  }
  *crc_out = crc;
  return cudaSuccess;
}

}  // namespace sbbf
