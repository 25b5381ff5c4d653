# After pruning the A/B variants: full GPU suite and the headline bench.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2am_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2am_pytest.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2am_bench.json 2> gpurun_out/r2am_bench.err
