# Fused lookup sweep, spill-free nested-loop form: variants x pacing on config 4, then the parity subset.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cc_bench_$tag.json 2> gpurun_out/r2cc_bench_$tag.err
}
for v in 0 1 2 3; do
  run v${v}s0 4 SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=0
  run v${v}s2 4 SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=2
done
run v0s1 4 SBBF_FUSED_VARIANT=0 SBBF_FUSED_SLACK=1
run v0s3 4 SBBF_FUSED_VARIANT=0 SBBF_FUSED_SLACK=3
timeout 1200 python -m pytest tests -m gpu -q -x -k "blocked or config_full or random_parity or unaligned or regions or sharded or dist or config5" > gpurun_out/r2cc_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2cc_pytest.log
