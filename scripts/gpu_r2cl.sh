# Fused lookup sweep: one vs two sectors in flight per lane (6/8 vs 5/4 CTAs/SM), paced, config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env SBBF_FUSED_DEBUG=1 "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cl_bench_$tag.json 2> gpurun_out/r2cl_bench_$tag.err
}
for v in 0 1 2 3; do
  run v${v}s2 4 SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=2
done
run v2s3 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=3
run v3s3 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=3
run v2s0 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=0
