# Insert sweep: keys in 32-key blocks per segment (one 256-byte request), distributed by shuffle: bench + parity subset.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cx_bench_$tag.json 2> gpurun_out/r2cx_bench_$tag.err
}
run blk32
run blk32q4 SBBF_SEG_INS_Q=4
timeout 1200 python -m pytest tests -m gpu -q -x -k "blocked or config_full or golden_filters or random_parity or unaligned or foreign or idempot or concurrent or sharded or cuda_graph" > gpurun_out/r2cx_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2cx_pytest.log
