# Final tree of the round: full GPU suite (release), blocked/sharded subset on the debug library,
# headline bench + reference arm, world-1 sharded lines, per-phase ncu launch lists for config 4.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2cq_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2cq_pytest.log
SBBF_LIB=debug timeout 1500 python -m pytest tests -m gpu -q -x -k "blocked or unaligned or foreign or config_small or two_level or sharded_filter_world1 or fused_route or multi_shard" > gpurun_out/r2cq_pytest_debug.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2cq_pytest_debug.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2cq_ref.json 2> gpurun_out/r2cq_ref.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2cq_bench.json 2> gpurun_out/r2cq_bench.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r2cq_cfg5_world1.json 2> gpurun_out/r2cq_cfg5_world1.err
timeout 900 python bench.py --sharded --config 4 --steps 5 --warmup 3 > gpurun_out/r2cq_sharded_cfg4_world1.json 2> gpurun_out/r2cq_sharded_cfg4_world1.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for ph in insert lookup; do
  timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/r2cq_launch_4_${ph}.csv python scripts/profile_phase.py 4 $ph \
    > gpurun_out/r2cq_launch_4_${ph}.log 2>&1
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2cq_smoke.log 2>&1
