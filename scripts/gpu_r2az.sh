set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "blocked or config_full or golden_filters or random_parity or config5 or sharded or graph" > gpurun_out/r2az_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2az_pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2az_bench_$tag.json 2> gpurun_out/r2az_bench_$tag.err; }
run new
run new2
