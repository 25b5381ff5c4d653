#!/bin/bash
# Round-1h evidence (end of round 1): the default bench line, the reference
# arm, the config-2 launch list of the bench command (gpu__time_duration
# only) and one ncu --set full capture each of the headline lookup and
# insert kernels. Every ncu pass runs only after its command exited 0
# without ncu.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r1h_smi.txt
timeout 600 python bench.py > gpurun_out/r1h_bench_line.json 2> gpurun_out/r1h_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r1h_bench_reference_line.json 2> gpurun_out/r1h_bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --extra , --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r1h_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1h_launches_cfg2.csv $CMD > gpurun_out/r1h_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"find_whole_kernel|insert_wide_kernel" -s 6 -c 2 -o gpurun_out/r1h_prof_cfg2 \
  $CMD > gpurun_out/r1h_ncu_full.log 2>&1
ls -la gpurun_out | tail -12
