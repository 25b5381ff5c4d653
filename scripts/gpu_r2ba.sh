# Session re-entry check: full GPU suite on HEAD, headline bench + reference arm.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2ba_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2ba_pytest.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2ba_ref.json 2> gpurun_out/r2ba_ref.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2ba_bench.json 2> gpurun_out/r2ba_bench.err
