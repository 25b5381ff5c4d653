# Tile inserts: parity under SBBF_INSERT_TILES=1, insert-phase timing, bench,
# per-kernel ncu times.
set -x
mkdir -p gpurun_out
SBBF_INSERT_TILES=1 timeout 300 python scripts/insert_dup_probe.py 3 > gpurun_out/r2ae_dup_tiles.log 2>&1
SBBF_INSERT_TILES=1 timeout 900 python -m pytest tests -m gpu -q -x -k "tile or blocked or config_full or random_parity or golden_filters or config_small" > gpurun_out/r2ae_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ae_pytest.log
SBBF_INSERT_TILES=1 timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ae_bench_tiles.json 2> gpurun_out/r2ae_bench_tiles.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
SBBF_INSERT_TILES=1 timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2ae_launch_tiles_insert.csv python scripts/profile_phase.py 4 insert > /dev/null 2>&1
