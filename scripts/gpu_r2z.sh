# A/B on top of TMA scatter without the side-stream pipeline: TMA unpermute,
# lean insert segment kernels.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env SBBF_SCATTER_TMA=1 SBBF_BLOCKED_PIPELINE=0 "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2z_bench_$tag.json 2> gpurun_out/r2z_bench_$tag.err
}
run tma 4
run ut 4 SBBF_UNPERM_TMA=1
run l8 4 SBBF_SEG_INS_Q=6008
run l6 4 SBBF_SEG_INS_Q=6006
run l4 4 SBBF_SEG_INS_Q=6004
run ut_l8 4 SBBF_UNPERM_TMA=1 SBBF_SEG_INS_Q=6008
SBBF_SCATTER_TMA=1 SBBF_BLOCKED_PIPELINE=0 SBBF_UNPERM_TMA=1 SBBF_SEG_INS_Q=6008 timeout 900 python -m pytest tests -m gpu -q -x -k "blocked or config_full or golden_filters or random_parity" > gpurun_out/r2z_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2z_pytest.log
