# Round-1 final evidence: bench lines (ours + reference arm), the config-2
# launch list, and ncu --set full captures of the top kernels.
set -x
python bench.py > gpurun_out/bench_final.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --extra , --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain2b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_r1b.csv $CMD > gpurun_out/ncu_l2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:find_pipe -s 3 -c 1 -o gpurun_out/prof_find_pipe_cfg2 $CMD > gpurun_out/ncu_fp2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:insert_wide -s 3 -c 1 -o gpurun_out/prof_insert_wide_cfg2 $CMD > gpurun_out/ncu_iw2.log 2>&1
python scripts/profile_blocked.py 4 find 3 2 > gpurun_out/pbf4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bucket_scatter|probe_grouped" -c 2 -o gpurun_out/prof_blocked_find_cfg4 python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/ncu_bf4.log 2>&1
ls -la gpurun_out | tail -5
