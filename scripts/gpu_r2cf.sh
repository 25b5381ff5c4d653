# Fused lookup sweep: smaller slices (16 / 8 MiB) with pacing and next-slice prefetch, config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cf_bench_$tag.json 2> gpurun_out/r2cf_bench_$tag.err
}
for mb in 16 8; do
 for v in 3 2; do
   run m${mb}v${v}s2p0 4 SBBF_SLICE_MB=$mb SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=0
   run m${mb}v${v}s2p1 4 SBBF_SLICE_MB=$mb SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=1
   run m${mb}v${v}s1p1 4 SBBF_SLICE_MB=$mb SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=1 SBBF_FUSED_PREFETCH=1
 done
done
