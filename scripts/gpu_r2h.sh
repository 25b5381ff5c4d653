set -x
mkdir -p gpurun_out
timeout 120 scripts/bin/microbench_l2res 0x80000000 > gpurun_out/r2h_l2res.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2h_l2res_ncu.csv scripts/bin/microbench_l2res 0x80000000 > /dev/null 2>&1
for sl in 2 3; do
  SBBF_SWEEP_SLACK=$sl timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2h_bench_sl$sl.json 2> gpurun_out/r2h_bench_sl$sl.err
done
SBBF_SWEEP_SLACK=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2h_launch_4_insert.csv python scripts/profile_blocked.py 4 insert 6 1 > /dev/null 2>&1
