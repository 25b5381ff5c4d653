# Fused lookup sweep with slice pacing: A/B on config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env SBBF_FUSED_DEBUG=1 "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cb_bench_$tag.json 2> gpurun_out/r2cb_bench_$tag.err
}
run s2 4 SBBF_FUSED_SLACK=2
run s1 4 SBBF_FUSED_SLACK=1
run s3 4 SBBF_FUSED_SLACK=3
run s2pf 4 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=1
run s1pf 4 SBBF_FUSED_SLACK=1 SBBF_FUSED_PREFETCH=1
run s2w2 4 SBBF_FUSED_SLACK=2 SBBF_FUSED_W=2
