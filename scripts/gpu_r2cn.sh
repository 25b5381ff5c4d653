# Fused lookup sweep as the default: full GPU suite (release), blocked subset on the debug
# library (SBBF_DCHECK), headline bench + reference arm, per-phase ncu launch lists for
# config 4 (traffic.json), one --set full capture of the fused sweep.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2cn_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2cn_pytest.log
SBBF_LIB=debug timeout 1500 python -m pytest tests -m gpu -q -x -k "blocked or unaligned or foreign or config_small or two_level or sharded_filter_world1" > gpurun_out/r2cn_pytest_debug.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2cn_pytest_debug.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2cn_ref.json 2> gpurun_out/r2cn_ref.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2cn_bench.json 2> gpurun_out/r2cn_bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for cid in 4; do
  for ph in insert lookup; do
    timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/r2cn_launch_${cid}_${ph}.csv python scripts/profile_phase.py $cid $ph \
      > gpurun_out/r2cn_launch_${cid}_${ph}.log 2>&1
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sweep_find" -c 1 -o gpurun_out/r2cn_sweep_find -f python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2cn_ncu.log 2>&1
