# Round 2: per-phase ncu launch lists (duration, DRAM bytes, L2 hit rate) of
# every kernel bench.py's insert and lookup phases launch, configs 2/3/4,
# plus one --set full capture of the config-4 lookup segment kernel.
# Summarised here by scripts/traffic.py into profiles/traffic.json.
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for cid in 2 3 4; do
  for ph in insert lookup; do
    timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/r2_launch_${cid}_${ph}.csv python scripts/profile_phase.py $cid $ph \
      > gpurun_out/r2_launch_${cid}_${ph}.log 2>&1
  done
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:segment_kernel -c 1 -o gpurun_out/r2_seg_lookup python scripts/profile_phase.py 4 lookup \
  > gpurun_out/r2_seg_lookup.log 2>&1
