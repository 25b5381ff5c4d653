# New defaults (TMA partition + unpermute, no lookup pipeline): full GPU suite,
# headline bench + reference arm, per-phase ncu launch lists (traffic.json),
# ncu --set full of the TMA partition.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2af_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2af_pytest.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2af_ref.json 2> gpurun_out/r2af_ref.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2af_bench.json 2> gpurun_out/r2af_bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for cid in 3 4; do
  for ph in insert lookup; do
    timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/r2af_launch_${cid}_${ph}.csv python scripts/profile_phase.py $cid $ph \
      > gpurun_out/r2af_launch_${cid}_${ph}.log 2>&1
  done
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:chunk_scatter_tma -c 1 -o gpurun_out/r2af_scatter_tma python scripts/profile_phase.py 4 lookup \
  > gpurun_out/r2af_scatter_tma.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:unpermute_tma -c 1 -o gpurun_out/r2af_unperm_tma python scripts/profile_phase.py 4 lookup \
  > gpurun_out/r2af_unperm_tma.log 2>&1
