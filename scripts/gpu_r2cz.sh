# Fused sweep probes with the L2 evict-last hint (the slot stream keeps its evict-first hint), config 4.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cz_bench_$tag.json 2> gpurun_out/r2cz_bench_$tag.err
}
run base SBBF_KEY_LD=0
run last SBBF_KEY_LD=10
run last_s3 SBBF_KEY_LD=10 SBBF_FUSED_SLACK=3
