# Cache policy of the sweeps' staged-key loads: evict-first hint (default) vs no hint vs ld.global.cs, config 4.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cy_bench_$tag.json 2> gpurun_out/r2cy_bench_$tag.err
}
run ld0 SBBF_KEY_LD=0
run ld1 SBBF_KEY_LD=1
run ld2 SBBF_KEY_LD=2
