set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2o_bench_$tag.json 2> gpurun_out/r2o_bench_$tag.err
}
run c4base 4
run c4p1 4 SBBF_PART_PER_SM=1
run c4p1s20 4 SBBF_PART_PER_SM=1 SBBF_SEG_SMEM_KB=20
run c4np 4 SBBF_BLOCKED_PIPELINE=0
run c3 3
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2o_launch_3_lookup.csv python scripts/profile_phase.py 3 lookup > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/r2o_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2o_pytest.log
