// sbbf_image.cu — FilterImage v1 on device: CRC-32 (IEEE, reflected 0xEDB88320)
// of the block array computed on the GPU (persist.cpp:64-70 is the
// byte-serial reference), for sbbf_gpu_serialize / sbbf_gpu_deserialize /
// sbbf_gpu_image_crc (image layout: persist.hpp:14-30).
//
// Parallel CRC: CRC is linear over GF(2), so crc(A||B) =
// crc(A) * x^(8|B|) mod P  xor  crc(B) (the "combine" identity zlib's
// crc32_combine uses). Each CTA walks a contiguous run of 64 KiB segments:
// a segment is loaded with coalesced 16-byte loads into a padded shared-memory
// layout (no bank conflicts when every thread reads its own 256-byte piece),
// every thread CRCs its piece with slicing-by-8 tables in smem and folds it
// into a per-thread Horner accumulator; one scaling per thread and an XOR
// reduction give the CTA's CRC, and the host combines the few hundred
// per-CTA values.
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
constexpr uint32_t kSegmentSmem = kSegment + kSegment / 64;  // + one pad word per 256-byte piece

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
__host__ __device__ uint32_t xpow8n(uint64_t nbytes) {
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
  uint32_t shift[kCrcThreads];  // x^(8 * (kSegment - kPiece * (t + 1))): piece t to its segment's end
  uint32_t segment;             // x^(8 * kSegment)
};

// Shared-memory word index of segment word w: one pad word per 64 words
// (one thread's 256-byte piece), so the 32 lanes of a warp reading word j of
// their own pieces hit 32 different banks.
__device__ __forceinline__ uint32_t padded(uint32_t w) { return w + (w >> 6); }

// CTA c CRCs the contiguous segments [c*per, (c+1)*per) and writes the CRC of
// that whole range to seg_crc[c]; the host combines the per-CTA values.
//
// CRC-32 is affine in the message, so crc(A || B) = x^(8|B|) * crc(A) ^
// crc(B) (the zlib combine; multmodp is the product mod P). Thread t keeps a
// Horner accumulator of its piece CRCs over the full segments, acc = x^(8 *
// kSegment) * acc ^ crc(piece) (a constant multiplier, applied with four
// 256-entry byte tables), and scales it once by x^(8 * bytes after its
// piece); the CTA XOR-reduces the results. No per-segment tree or serial
// combine. A ragged last segment (the image end) is scaled directly.
__global__ void __launch_bounds__(kCrcThreads) crc_segments_kernel(const uint8_t* __restrict__ data,
                                                                   uint64_t bytes, uint64_t per, CrcOps ops,
                                                                   uint32_t* __restrict__ seg_crc) {
  __shared__ uint32_t table[8][256];
  __shared__ uint32_t horner[4][256];  // horner[k][b] = x^(8 * kSegment) * (b << 8k)
  __shared__ uint32_t red[kCrcThreads / 32];
  extern __shared__ __align__(16) uint32_t seg[];  // kSegmentSmem bytes: the padded 64 KiB segment
  const uint32_t t = threadIdx.x;
  // slicing-by-8 tables (table[0] is the byte-serial table of persist.cpp:15-28)
  {
    uint32_t c = t;
    for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
    table[0][t] = c;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) horner[k][t] = multmodp(ops.segment, t << (8 * k));
  __syncthreads();
  for (int k = 1; k < 8; ++k) {
    const uint32_t prev = table[k - 1][t];
    table[k][t] = (prev >> 8) ^ table[0][prev & 0xFFu];
    __syncthreads();
  }
  const uint64_t nseg = (bytes + kSegment - 1) / kSegment;
  const uint64_t s0 = static_cast<uint64_t>(blockIdx.x) * per;
  const uint64_t s1 = s0 + per < nseg ? s0 + per : nseg;
  // Each thread holds its 16 16-byte words of the segment in registers: the
  // next segment's loads are issued before this segment's CRC work, so HBM
  // latency hides behind the table lookups (block arrays are 32-byte
  // multiples, so len is a multiple of 16).
  constexpr uint32_t kVecs = kSegment / 16 / kCrcThreads;
  uint4 x[kVecs];
  auto load = [&](uint64_t sg) {
    const uint64_t off = sg * kSegment;
    const uint32_t nv = static_cast<uint32_t>((bytes - off < kSegment ? bytes - off : kSegment) / 16);
    const uint4* src = reinterpret_cast<const uint4*>(data + off);
#pragma unroll
    for (uint32_t j = 0; j < kVecs; ++j) {
      const uint32_t v = t + j * kCrcThreads;
      if (v < nv) x[j] = __ldg(src + v);
    }
  };
  if (s0 < s1) load(s0);
  uint32_t acc = 0;       // Horner accumulator over the full segments
  uint32_t ragged = 0;    // this piece's share of a ragged last segment
  uint32_t last_len = 0;  // that segment's length (0: none)
  for (uint64_t sg = s0; sg < s1; ++sg) {
    const uint64_t off = sg * kSegment;
    const uint32_t len = static_cast<uint32_t>(bytes - off < kSegment ? bytes - off : kSegment);
#pragma unroll
    for (uint32_t j = 0; j < kVecs; ++j) {
      const uint32_t v = t + j * kCrcThreads;
      if (v < len / 16) {
        const uint32_t w = 4 * v;
        seg[padded(w)] = x[j].x;
        seg[padded(w + 1)] = x[j].y;
        seg[padded(w + 2)] = x[j].z;
        seg[padded(w + 3)] = x[j].w;
      }
    }
    __syncthreads();
    if (sg + 1 < s1) load(sg + 1);
    // standard CRC-32 of this thread's 256-byte piece, 8 bytes per step
    const uint32_t pb = t * kPiece;
    const uint32_t plen = pb >= len ? 0 : (len - pb < kPiece ? len - pb : kPiece);
    uint32_t c = 0xFFFFFFFFu;
    for (uint32_t i = 0; i + 8 <= plen; i += 8) {
      const uint32_t wi = (pb + i) >> 2;
      const uint32_t lo = seg[padded(wi)] ^ c;
      const uint32_t hi = seg[padded(wi + 1)];
      c = table[7][lo & 0xFF] ^ table[6][(lo >> 8) & 0xFF] ^ table[5][(lo >> 16) & 0xFF] ^ table[4][lo >> 24] ^
          table[3][hi & 0xFF] ^ table[2][(hi >> 8) & 0xFF] ^ table[1][(hi >> 16) & 0xFF] ^ table[0][hi >> 24];
    }
    c ^= 0xFFFFFFFFu;  // an empty piece has CRC 0
    if (len == kSegment) {
      acc = horner[0][acc & 0xFF] ^ horner[1][(acc >> 8) & 0xFF] ^ horner[2][(acc >> 16) & 0xFF] ^
            horner[3][acc >> 24] ^ c;
    } else {
      ragged = plen ? multmodp(xpow8n(len - pb - plen), c) : 0;
      last_len = len;
    }
    __syncthreads();  // seg[] is rewritten by the next segment
  }
  uint32_t v = acc ? multmodp(ops.shift[t], acc) : 0;
  if (last_len) v = (v ? multmodp(xpow8n(last_len), v) : 0) ^ ragged;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, d);
  if ((t & 31) == 0) red[t >> 5] = v;
  __syncthreads();
  if (t == 0 && s0 < s1) {
    uint32_t r = 0;
#pragma unroll
    for (int w = 0; w < kCrcThreads / 32; ++w) r ^= red[w];
    seg_crc[blockIdx.x] = r;
  }
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
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t ctas_max = static_cast<uint64_t>(sms) * 2;  // ~83 KB smem per CTA
  const uint64_t per = (nseg + ctas_max - 1) / ctas_max;
  const uint64_t ctas = (nseg + per - 1) / per;
  // the staging copy moves 16-byte words: images are 32 * nb bytes
  if (bytes % 16 != 0 || reinterpret_cast<uintptr_t>(d_data) % 16 != 0) return cudaErrorInvalidValue;
  static const cudaError_t attr =
      cudaFuncSetAttribute(crc_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSegmentSmem);
  if (attr != cudaSuccess) return attr;
  CrcOps ops;
  for (uint32_t t = 0; t < kCrcThreads; ++t) ops.shift[t] = xpow8n(kSegment - kPiece * (t + 1));
  ops.segment = xpow8n(kSegment);
  uint32_t* d_seg = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_seg), ctas * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  note_launch();
  crc_segments_kernel<<<static_cast<unsigned>(ctas), kCrcThreads, kSegmentSmem, s>>>(static_cast<const uint8_t*>(d_data),
                                                                        bytes, per, ops, d_seg);
  e = cudaGetLastError();
  std::vector<uint32_t> part(ctas);
  if (e == cudaSuccess) e = cudaMemcpyAsync(part.data(), d_seg, ctas * sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d_seg, s);
  if (e != cudaSuccess) return e;
  const uint64_t range = per * kSegment;
  const uint32_t op_full = xpow8n(range);
  uint32_t crc = part[0];
  for (uint64_t i = 1; i < ctas; ++i) {
    const uint64_t len = (i == ctas - 1) ? bytes - i * range : range;
    crc = multmodp(len == range ? op_full : xpow8n(len), crc) ^ part[i];
  }
  *crc_out = crc;
  return cudaSuccess;
}

}  // namespace sbbf
