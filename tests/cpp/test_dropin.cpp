// C++ drop-in test: the reference's call pattern (tools/harness.cpp:160-171:
// construct, add_hashes(span), find_hashes(span, uint8_t*)) against
// sbbf::gpu::SplitBlockFilter, checked byte-for-byte with the oracle.
// Built and run by tests/test_cpp_dropin.py.
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

#include "sbbf_gpu.hpp"

extern "C" {
void oracle_gen_splitmix(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out);
void oracle_add_hashes(uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes, uint64_t n);
void oracle_find_hashes(const uint32_t* blocks, uint64_t num_buckets, const uint64_t* hashes,
                        uint64_t n, uint8_t* results);
uint32_t oracle_image_crc(const uint32_t* blocks, uint64_t num_buckets, uint32_t hasher_id);
}

#define REQUIRE(c)                                                     \
  do {                                                                 \
    if (!(c)) {                                                        \
      std::fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__);   \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main() {
  // config 1: 100k keys (splitmix64 seed 1) into 4096 blocks
  const uint64_t nb = 4096;
  std::vector<uint64_t> ins(100000), non(1000000);
  oracle_gen_splitmix(1, 0, ins.size(), ins.data());
  oracle_gen_splitmix(2, 0, non.size(), non.data());

  sbbf::gpu::SplitBlockFilter f(nb);
  REQUIRE(f.num_buckets() == nb && f.size_bytes() == nb * 32 && f.hasher_id() == 0);
  f.add_hashes(ins);
  const auto blocks = f.blocks();

  std::vector<uint32_t> want(nb * 8, 0);
  oracle_add_hashes(want.data(), nb, ins.data(), ins.size());
  REQUIRE(std::memcmp(blocks.data(), want.data(), nb * 32) == 0);
  REQUIRE(oracle_image_crc(reinterpret_cast<const uint32_t*>(blocks.data()), nb, 0) == 0xe34f8befu);

  std::vector<uint8_t> got(non.size()), ref(non.size());
  f.find_hashes(non, got.data());
  oracle_find_hashes(want.data(), nb, non.data(), non.size(), ref.data());
  REQUIRE(got == ref);
  uint64_t fp = 0;
  for (uint8_t r : got) fp += r;
  REQUIRE(fp == 10190);  // SURVEY.md §8(c) golden FP count
  const auto mem = f.find_hashes(ins);
  for (uint8_t r : mem) REQUIRE(r == 1);

  // error behaviour mirrors filter.cpp:160-162
  bool threw = false;
  try {
    sbbf::gpu::SplitBlockFilter bad(0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);

  // from_blocks / operator== / single-key ops
  auto g = sbbf::gpu::SplitBlockFilter::from_blocks(blocks);
  REQUIRE(g == f);
  sbbf::gpu::SplitBlockFilter one(1);
  one.add_hash(0);
  REQUIRE(one.find_hash(0));
  const auto one_blocks = one.blocks();  // keep the temporary alive for the loop
  for (uint32_t lane : one_blocks[0].lanes) REQUIRE(lane == 1u);
  // persist.hpp mirror: serialize -> deserialize round trip, CRC trailer,
  // and the reference's error codes (persist_test.cpp:140-193)
  const auto img = sbbf::gpu::serialize(f);
  REQUIRE(img.size() == 17 + nb * 32 + 4);
  const uint32_t trailer = img[img.size() - 4] | (img[img.size() - 3] << 8) | (img[img.size() - 2] << 16) |
                           (static_cast<uint32_t>(img[img.size() - 1]) << 24);
  REQUIRE(trailer == 0xe34f8befu);
  auto back = sbbf::gpu::deserialize(img);
  REQUIRE(back == f);
  auto bad = img;
  bad[100] ^= 1;
  bool checksum = false;
  try {
    sbbf::gpu::deserialize(bad);
  } catch (const sbbf::gpu::PersistError& e) {
    checksum = e.code() == sbbf::gpu::PersistErrc::kBadChecksum;
  }
  REQUIRE(checksum);
  bool io = false;
  try {
    sbbf::gpu::load_filter("/nonexistent/dir/f.sbbf");
  } catch (const sbbf::gpu::PersistError& e) {
    io = e.code() == sbbf::gpu::PersistErrc::kIo;
  }
  REQUIRE(io);
  // the C++ sharded layer over a 1-rank NCCL communicator (skipped when the
  // machine has no NCCL: sbbf_dist_* report SBBF_ENODEV then)
  unsigned char uid[128];
  if (sbbf_dist_unique_id(uid) == SBBF_OK) {
    void* comm = nullptr;
    REQUIRE(sbbf_dist_comm_init(uid, 1, 0, 0, &comm) == SBBF_OK);
    sbbf_dist_t* dist = nullptr;
    REQUIRE(sbbf_dist_create(comm, nb, 1u << 20, 0, &dist) == SBBF_OK);
    uint64_t* d_keys = nullptr;
    uint8_t* d_res = nullptr;
    REQUIRE(cudaMalloc(&d_keys, non.size() * 8) == cudaSuccess);
    REQUIRE(cudaMalloc(&d_res, non.size()) == cudaSuccess);
    REQUIRE(cudaMemcpy(d_keys, ins.data(), ins.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess);
    REQUIRE(sbbf_dist_insert(dist, d_keys, ins.size(), nullptr) == SBBF_OK);
    REQUIRE(cudaMemcpy(d_keys, non.data(), non.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess);
    REQUIRE(sbbf_dist_find(dist, d_keys, non.size(), d_res, nullptr) == SBBF_OK);
    std::vector<uint8_t> dres(non.size());
    REQUIRE(cudaMemcpy(dres.data(), d_res, non.size(), cudaMemcpyDeviceToHost) == cudaSuccess);
    REQUIRE(dres == ref);
    std::vector<uint32_t> whole(nb * 8);
    REQUIRE(sbbf_dist_gather(dist, whole.data(), 0) == SBBF_OK);
    REQUIRE(whole == want);
    cudaFree(d_keys);
    cudaFree(d_res);
    REQUIRE(sbbf_dist_destroy(dist) == SBBF_OK);
    {  // the RAII wrapper
      sbbf::gpu::ShardedFilter sf(comm, nb, 1u << 20);
      REQUIRE(sf.rank() == 0 && sf.world() == 1);
      REQUIRE(cudaMalloc(&d_keys, ins.size() * 8) == cudaSuccess);
      REQUIRE(cudaMemcpy(d_keys, ins.data(), ins.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess);
      sf.add_hashes_device(d_keys, ins.size());
      const auto whole_blocks = sf.blocks();
      REQUIRE(std::memcmp(whole_blocks.data(), want.data(), nb * 32) == 0);
      cudaFree(d_keys);
    }
    REQUIRE(sbbf_dist_comm_destroy(comm) == SBBF_OK);
    std::printf("cpp sharded layer (world 1) ok\n");
  }
  std::printf("cpp drop-in ok: crc 0xe34f8bef, %llu false positives\n", (unsigned long long)fp);
  return 0;
}
