# Fused sweep with the slot ring (slots copied into shared memory a run ahead by cp.async): A/B + parity subset.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env SBBF_FUSED_DEBUG=1 "$@" timeout 300 python bench.py --config 4 --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cu_bench_$tag.json 2> gpurun_out/r2cu_bench_$tag.err
}
run v0 SBBF_FUSED_VARIANT=0
run v2 SBBF_FUSED_VARIANT=2
run v3 SBBF_FUSED_VARIANT=3
run v2s0 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=0
run v2s3 SBBF_FUSED_VARIANT=2 SBBF_FUSED_SLACK=3
SBBF_FUSED_VARIANT=2 timeout 1200 python -m pytest tests -m gpu -q -x -k "blocked or config_full or random_parity or unaligned or foreign or sharded or dist or config5 or cuda_graph" > gpurun_out/r2cu_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2cu_pytest.log
