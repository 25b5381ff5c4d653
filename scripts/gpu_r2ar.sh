set -x
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ar_bench_$tag.json 2> gpurun_out/r2ar_bench_$tag.err; }
run r28
run r29 SBBF_BLOCKED_ROUND_LOG2=29
run r30 SBBF_BLOCKED_ROUND_LOG2=30
run r31 SBBF_BLOCKED_ROUND_LOG2=31
