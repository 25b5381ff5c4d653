# Fused sweep on the sharded layer's multi-region calls; side-stream lookup pipeline removed:
# sharded / blocked tests (release + debug library), world-1 sharded bench lines (config 5 sample, config 4).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "blocked or sharded or dist or route or foreign or config5 or cuda_graph or unaligned" > gpurun_out/r2cp_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2cp_pytest.log
SBBF_LIB=debug timeout 1500 python -m pytest tests -m gpu -q -x -k "blocked or foreign or fused_route or sharded_filter_world1 or multi_shard" > gpurun_out/r2cp_pytest_debug.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2cp_pytest_debug.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r2cp_cfg5_world1.json 2> gpurun_out/r2cp_cfg5_world1.err
timeout 900 python bench.py --sharded --config 4 --steps 5 --warmup 3 > gpurun_out/r2cp_sharded_cfg4_world1.json 2> gpurun_out/r2cp_sharded_cfg4_world1.err
