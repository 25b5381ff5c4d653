# ncu launch lists of the blocked path (kernel durations, DRAM bytes, L2 hit rate)
set -x
for args in ${PB_ARGS:-"4 insert 6" "4 find 3"}; do :; done
for args in "4 insert 6" "4 find 3" "3 find 3"; do
  tag=$(echo $args | tr ' ' '_')
  python scripts/profile_blocked.py $args 2 > gpurun_out/pb_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/pb_launch_$tag.csv python scripts/profile_blocked.py $args 2 > gpurun_out/pb_ncu_$tag.log 2>&1
done
