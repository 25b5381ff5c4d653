set -x
python scripts/sweep.py sectors > gpurun_out/sweep_sectors.log 2>&1
python scripts/sweep.py variants > gpurun_out/sweep_variants.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --extra , --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_l2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:find_global -s 3 -c 1 -o gpurun_out/prof_find_cfg2 $CMD > gpurun_out/ncu_f2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:insert_lane8 -s 3 -c 1 -o gpurun_out/prof_insert_cfg2 $CMD > gpurun_out/ncu_i2.log 2>&1
CMD4="python bench.py --config 4 --steps 1 --warmup 3 --extra , --no-cpu-baseline --no-e2e"
$CMD4 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:find_global -s 3 -c 1 -o gpurun_out/prof_find_cfg4 $CMD4 > gpurun_out/ncu_f4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:insert_lane8 -s 20 -c 1 -o gpurun_out/prof_insert_cfg4 $CMD4 > gpurun_out/ncu_i4.log 2>&1
ls -la gpurun_out
