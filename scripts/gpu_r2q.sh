set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2q_bench_$tag.json 2> gpurun_out/r2q_bench_$tag.err
}
run c4q4 4
run c4q2 4 SBBF_SEG_INS_Q=2
run c4q8 4 SBBF_SEG_INS_Q=8
run c3s0 3
run c3s1 3 SBBF_SPLIT_VARIANT=1
run c3s2 3 SBBF_SPLIT_VARIANT=2
