# Slot-ring variant of the fused sweep after the long-run tail fix: parity + timing.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cv_bench_$tag.json 2> gpurun_out/r2cv_bench_$tag.err
}
run v2 SBBF_FUSED_VARIANT=2
run v3 SBBF_FUSED_VARIANT=3
run v0w5 SBBF_FUSED_VARIANT=0 SBBF_FUSED_W=5
SBBF_FUSED_VARIANT=2 timeout 900 python -m pytest tests -m gpu -q -x -k "blocked or config_full or unaligned or foreign or cuda_graph" > gpurun_out/r2cv_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2cv_pytest.log
