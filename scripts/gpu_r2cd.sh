# ncu launch lists (duration, DRAM bytes, L2 hit rate) of the fused lookup sweep, 6 and 8 CTAs/SM.
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for v in 3 2; do
  SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=0 ncu --metrics $M --clock-control none -k regex:"sweep_find|chunk_scatter" --csv --log-file gpurun_out/r2cd_launch_v$v.csv python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2cd_ncu_v$v.log 2>&1
done
