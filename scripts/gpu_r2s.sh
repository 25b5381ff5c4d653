# Round 2 re-entry: full GPU suite, headline bench + reference arm, per-phase
# ncu traffic launch lists for configs 2/3/4 (roofline.traffic).
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r2s_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2s_pytest.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
bash scripts/gpu_profile_r2_traffic.sh
