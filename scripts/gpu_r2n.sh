set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r2n_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2n_pytest.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2n_ref.json 2> gpurun_out/r2n_ref.err
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
