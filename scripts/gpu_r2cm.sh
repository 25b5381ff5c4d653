# Fused lookup sweep: L2 fill size of probe misses (sector / 128 B / 256 B), config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cm_bench_$tag.json 2> gpurun_out/r2cm_bench_$tag.err
}
for f in 1 2; do
  run v0s2f$f 4 SBBF_FUSED_VARIANT=0 SBBF_FUSED_SLACK=2 SBBF_FUSED_FILL=$f
  run v1s2f$f 4 SBBF_FUSED_VARIANT=1 SBBF_FUSED_SLACK=2 SBBF_FUSED_FILL=$f
  run v2s2f$f 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=2 SBBF_FUSED_FILL=$f
done
run v0s0f1 4 SBBF_FUSED_VARIANT=0 SBBF_FUSED_SLACK=0 SBBF_FUSED_FILL=1
run v0s3f1 4 SBBF_FUSED_VARIANT=0 SBBF_FUSED_SLACK=3 SBBF_FUSED_FILL=1
