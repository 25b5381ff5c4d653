set -x
mkdir -p gpurun_out
SBBF_INSERT_TILES=1 SBBF_TILE_APPLY=1 timeout 300 python scripts/insert_dup_probe.py 3 > gpurun_out/r2as_dup_v1.log 2>&1
SBBF_INSERT_TILES=1 SBBF_TILE_APPLY=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_insert or blocked_path_skew" > gpurun_out/r2as_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2as_pytest.log
SBBF_INSERT_TILES=1 SBBF_TILE_APPLY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2as_launch.csv python scripts/profile_phase.py 4 insert > /dev/null 2>&1
