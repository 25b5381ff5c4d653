set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2i_bench_$tag.json 2> gpurun_out/r2i_bench_$tag.err
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2i_launch_$tag.csv python scripts/profile_blocked.py 4 find 3 1 > /dev/null 2>&1
}
run s1p0 SBBF_SWEEP_SLACK=1 SBBF_SWEEP_PREFETCH=0
run s2p0 SBBF_SWEEP_SLACK=2 SBBF_SWEEP_PREFETCH=0
run s1p0m16 SBBF_SWEEP_SLACK=1 SBBF_SWEEP_PREFETCH=0 SBBF_SLICE_MB=16
run s2p0m16 SBBF_SWEEP_SLACK=2 SBBF_SWEEP_PREFETCH=0 SBBF_SLICE_MB=16
run s1p1m16 SBBF_SWEEP_SLACK=1 SBBF_SWEEP_PREFETCH=1 SBBF_SLICE_MB=16
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q -x -k "world_gt1 or world1 or c_abi" > gpurun_out/r2i_pytest_dist.log 2>&1
