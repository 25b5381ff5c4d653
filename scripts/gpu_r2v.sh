# A/B: L2 prefetch of the next step's filter lines in the config-4 segment
# kernels; L2 persisting window on config 3's range-split passes.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2v_bench_$tag.json 2> gpurun_out/r2v_bench_$tag.err
}
nvidia-smi -q | grep -i -A3 "persist" | head -20
run base 4
run ipf 4 SBBF_SEG_INS_Q=2004
run lpf 4 SBBF_SEG_LOOK_PF=1
run both 4 SBBF_SEG_INS_Q=2004 SBBF_SEG_LOOK_PF=1
run c3 3
run c3w64 3 SBBF_SPLIT_PERSIST_MB=64
run c3w48 3 SBBF_SPLIT_PERSIST_MB=48
run c3w96 3 SBBF_SPLIT_PERSIST_MB=96
