# ncu: does the next-slice bulk prefetch remove the sweep's demand misses? (DRAM bytes, L2 hit rate)
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
for t in "p0 SBBF_FUSED_PREFETCH=0" "p1 SBBF_FUSED_PREFETCH=1"; do
  set -- $t
  env SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 $2 ncu --metrics $M --clock-control none -k regex:"sweep_find" --csv --log-file gpurun_out/r2ch_launch_$1.csv python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2ch_ncu_$1.log 2>&1
done
