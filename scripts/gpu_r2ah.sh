# A/B: 2 probes/lane at 8 CTAs/SM (spilling) for config-4 lookups; config 3
# persisting window re-measured with more steps.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ah_bench_$tag.json 2> gpurun_out/r2ah_bench_$tag.err
}
run base 4
run q2x8 4 SBBF_SEG_LOOK_Q=3
run c3 3
run c3w64 3 SBBF_SPLIT_PERSIST_MB=64
run c3b 3
run c3w64b 3 SBBF_SPLIT_PERSIST_MB=64
