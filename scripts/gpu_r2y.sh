# A/B: TMA scatter without the side-stream pipeline; alternating sweeps.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2y_bench_$tag.json 2> gpurun_out/r2y_bench_$tag.err
}
run base 4 SBBF_SEG_ALTERNATE=0
run alt 4
run tma_np 4 SBBF_SCATTER_TMA=1 SBBF_BLOCKED_PIPELINE=0 SBBF_SEG_ALTERNATE=0
run tma_np_alt 4 SBBF_SCATTER_TMA=1 SBBF_BLOCKED_PIPELINE=0
run np 4 SBBF_BLOCKED_PIPELINE=0 SBBF_SEG_ALTERNATE=0
run tma_alt 4 SBBF_SCATTER_TMA=1
