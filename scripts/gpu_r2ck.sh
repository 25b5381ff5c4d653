# ncu: slice prefetch (per line) x next-run slot prefetch on the fused sweep: time, DRAM bytes, L2 hits.
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
for t in "p0k0 0 0" "p2k0 2 0" "p0k1 0 1" "p2k1 2 1" "p1k1 1 1"; do
  set -- $t
  env SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 SBBF_FUSED_PREFETCH=$2 SBBF_FUSED_KEYPF=$3 ncu --metrics $M --clock-control none -k regex:"sweep_find" -c 1 --csv --log-file gpurun_out/r2ck_launch_$1.csv python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2ck_ncu_$1.log 2>&1
done
