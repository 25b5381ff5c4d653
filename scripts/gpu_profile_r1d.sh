# Round-1d evidence: clean config-2 launch list (gpu__time_duration only) of
# the bench command, and ncu --set full captures of the blocked-path kernels.
set -x
CMD="python bench.py --steps 2 --warmup 3 --extra , --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain2c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_r1d.csv $CMD > gpurun_out/ncu_l2c.log 2>&1
python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/pbf4c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"chunk_scatter|segment_kernel|unpermute" -s 8 -c 3 -o gpurun_out/prof_blocked_find_r1d python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/ncu_bf4c.log 2>&1
ls -la gpurun_out | tail -3
