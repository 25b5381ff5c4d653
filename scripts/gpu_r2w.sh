# A/B: insert segment test loads through L1 (.ca, default) vs .cg vs .nc, and
# 4 CTAs/SM.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2w_bench_$tag.json 2> gpurun_out/r2w_bench_$tag.err
}
run base 4
run cg 4 SBBF_SEG_INS_Q=3004
run nc 4 SBBF_SEG_INS_Q=4004
run cg4 4 SBBF_SEG_INS_Q=5004
run base2 4
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for v in 4 3004 5004; do
  SBBF_SEG_INS_Q=$v timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv -k regex:segment_kernel -c 2 \
    --log-file gpurun_out/r2w_ins_$v.csv python scripts/profile_phase.py 4 insert > /dev/null 2>&1
done
