/*
 * sbbf_bench.h — roofline microbenchmarks (not part of the reference API).
 * They measure the random 32-byte-sector ceiling that bounds SBBF insert and
 * lookup: the denominators of bench.py's "fraction of the random-sector
 * roofline" (BASELINE.json metric).
 */
#ifndef SBBF_BENCH_H
#define SBBF_BENCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* n random 256-bit reads of d_buf (num_blocks * 32 bytes), block indices from
 * splitmix64(seed) in registers; d_sink receives up to 1024 words. */
int sbbf_bench_sector_read(const uint32_t* d_buf, uint64_t num_blocks, uint64_t n, uint64_t seed,
                           uint32_t* d_sink, void* stream);
/* n random 32-byte atomic-OR sector updates (4 threads per key, one red.global.or.b64
 * per lane pair: the insert kernels' pattern). */
int sbbf_bench_sector_red(uint32_t* d_buf, uint64_t num_blocks, uint64_t n, uint64_t seed,
                          void* stream);

/* Live per-kernel timing of the L2-blocked path (bench.py's dominant-kernel
 * roofline). enable != 0 starts recording a CUDA event pair around every
 * blocked-path launch group on its stream and clears the totals; 0 stops.
 * sbbf_bench_kernel_times synchronises the recorded events and returns the
 * summed milliseconds and launch-group counts per kind, up to n kinds:
 * 0 partition (chunk_scatter), 1 lookup probe sweep (sweep_find_kernel, or
 * segment_kernel in the unfused form), 2 insert sweep, 3 unpermute (unfused
 * lookups only), 4 tile insert (tile_scatter + tile_apply). */
int sbbf_bench_kernel_timing(int enable);
int sbbf_bench_kernel_times(double* ms, uint64_t* launches, int n);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
