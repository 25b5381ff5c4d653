# Fused lookup sweep: next slice pulled into L2 by cp.async copies (sequential HBM reads), config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2co_bench_$tag.json 2> gpurun_out/r2co_bench_$tag.err
}
run s2 4 SBBF_FUSED_SLACK=2
run s2pull 4 SBBF_FUSED_SLACK=2 SBBF_FUSED_PULL=1
run s1pull 4 SBBF_FUSED_SLACK=1 SBBF_FUSED_PULL=1
run v1s2pull 4 SBBF_FUSED_VARIANT=1 SBBF_FUSED_SLACK=2 SBBF_FUSED_PULL=1
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
SBBF_FUSED_SLACK=2 SBBF_FUSED_PULL=1 ncu --metrics $M --clock-control none -k regex:"sweep_find" -c 1 --csv --log-file gpurun_out/r2co_launch_pull.csv python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2co_ncu_pull.log 2>&1
