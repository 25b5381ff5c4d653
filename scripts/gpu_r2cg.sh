# Fused lookup sweep: own rounds over the whole batch; next-run slot L2 prefetch x pacing x slice prefetch, config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cg_bench_$tag.json 2> gpurun_out/r2cg_bench_$tag.err
}
run v3s0k0 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=0 SBBF_FUSED_KEYPF=0
run v3s0k1 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=0 SBBF_FUSED_KEYPF=1
run v3s2p0k1 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=0 SBBF_FUSED_KEYPF=1
run v3s2p1k1 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=1 SBBF_FUSED_KEYPF=1
run v3s1p1k1 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=1 SBBF_FUSED_PREFETCH=1 SBBF_FUSED_KEYPF=1
run v2s2p0k1 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=0 SBBF_FUSED_KEYPF=1
run v2s2p1k1 4 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=1 SBBF_FUSED_KEYPF=1
