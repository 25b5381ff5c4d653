# Fused lookup sweep: up to 8 chunks per warp (233M-key rounds), per-line next-slice prefetch, config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env SBBF_FUSED_DEBUG=1 "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ci_bench_$tag.json 2> gpurun_out/r2ci_bench_$tag.err
}
run v3s0 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=0
run v3s2p0 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=0
run v3s2p2 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=2
run v3s1p2 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=1 SBBF_FUSED_PREFETCH=2
run v2s2p0 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=0
run v2s2p2 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=2
run v3s2p0w6 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=0 SBBF_FUSED_W=6
