set -x
mkdir -p gpurun_out
timeout 120 scripts/bin/microbench_l2res 0x4000 > gpurun_out/r2k_l2res.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2k_l2res_ncu.csv scripts/bin/microbench_l2res 0x4000 > /dev/null 2>&1
SBBF_DIST_DEBUG=1 timeout 200 python scripts/dist_hooks_debug.py > gpurun_out/r2k_dist_debug.log 2>&1
