# round 2a: ncu launch lists (duration + DRAM bytes + L2 hit rate) of the
# config 3 / 4 lookup and insert paths, the traffic behind roofline.traffic
set -x
mkdir -p gpurun_out
for args in "4 insert 6" "4 find 3" "3 find 1" "3 insert 4"; do
  tag=$(echo $args | tr ' ' '_')
  python scripts/profile_blocked.py $args 2 > gpurun_out/r2a_pb_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_red.sum --clock-control none --csv --log-file gpurun_out/r2a_launch_$tag.csv python scripts/profile_blocked.py $args 2 > gpurun_out/r2a_ncu_$tag.log 2>&1
done
