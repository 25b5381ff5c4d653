# Final defaults: full GPU suite, headline bench + reference arm, per-phase
# ncu launch lists for configs 3/4 (traffic.json).
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2at_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2at_pytest.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2at_ref.json 2> gpurun_out/r2at_ref.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2at_bench.json 2> gpurun_out/r2at_bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for cid in 4; do
  for ph in insert lookup; do
    timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/r2at_launch_${cid}_${ph}.csv python scripts/profile_phase.py $cid $ph \
      > gpurun_out/r2at_launch_${cid}_${ph}.log 2>&1
  done
done
