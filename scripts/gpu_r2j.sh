set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2j_bench_$tag.json 2> gpurun_out/r2j_bench_$tag.err
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2j_launch_$tag.csv python scripts/profile_blocked.py 4 find 3 1 > /dev/null 2>&1
}
run old64 SBBF_SWEEP=0
run old64np SBBF_SWEEP=0 SBBF_BLOCKED_PIPELINE=0
run old16np SBBF_SWEEP=0 SBBF_BLOCKED_PIPELINE=0 SBBF_SEG_CHUNKS=16
run old32np SBBF_SWEEP=0 SBBF_BLOCKED_PIPELINE=0 SBBF_SEG_CHUNKS=32
run old16np16 SBBF_SWEEP=0 SBBF_BLOCKED_PIPELINE=0 SBBF_SEG_CHUNKS=16 SBBF_SLICE_MB=16
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q -x -k "world_gt1" > gpurun_out/r2j_pytest_dist.log 2>&1
