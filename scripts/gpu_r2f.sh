# round 2f: persistent sweep — parity (blocked tests, full configs 3/4) then a config-4 bench A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "blocked or config_full or graph or config_small" > gpurun_out/r2f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f_pytest.log
timeout 300 python bench.py --config 4 --extra "" --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2f_bench_sweep.json 2> gpurun_out/r2f_bench_sweep.err
SBBF_SWEEP=0 timeout 300 python bench.py --config 4 --extra "" --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2f_bench_old.json 2> gpurun_out/r2f_bench_old.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2f_launch_4_find.csv python scripts/profile_blocked.py 4 find 3 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2f_launch_4_insert.csv python scripts/profile_blocked.py 4 insert 6 2 > /dev/null 2>&1
SBBF_SWEEP_PREFETCH=0 timeout 300 python bench.py --config 4 --extra "" --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2f_bench_nopf.json 2> gpurun_out/r2f_bench_nopf.err
