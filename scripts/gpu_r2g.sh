# round 2g: persistent sweep lockstep variants (slack) on config 4
set -x
mkdir -p gpurun_out
for sl in 0 1 2 3; do
  SBBF_SWEEP_DEBUG=1 SBBF_SWEEP_SLACK=$sl timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2g_bench_sl$sl.json 2> gpurun_out/r2g_bench_sl$sl.err
done
SBBF_SWEEP_SLACK=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2g_launch_4_find.csv python scripts/profile_blocked.py 4 find 3 1 > /dev/null 2>&1
SBBF_SWEEP_SLACK=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -c 2 -o gpurun_out/r2g_sweep python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2g_ncu_full.log 2>&1
