# Persistent tile apply: parity, insert-phase timing, per-kernel ncu times.
set -x
mkdir -p gpurun_out
SBBF_INSERT_TILES=1 timeout 300 python scripts/insert_dup_probe.py 3 > gpurun_out/r2ag_dup_tiles.log 2>&1
SBBF_INSERT_TILES=1 timeout 900 python -m pytest tests -m gpu -q -x -k "tile or blocked or config_full" > gpurun_out/r2ag_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ag_pytest.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
SBBF_INSERT_TILES=1 timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2ag_launch_tiles_insert.csv python scripts/profile_phase.py 4 insert > /dev/null 2>&1
