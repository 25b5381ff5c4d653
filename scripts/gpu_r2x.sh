# TMA chunk_scatter: parity under SBBF_SCATTER_TMA=1, then config-4/3 A/B.
set -x
mkdir -p gpurun_out
SBBF_SCATTER_TMA=1 timeout 900 python -m pytest tests -m gpu -q -x -k "blocked or random_parity or config_full or config5 or golden_filters or cuda_graph or sharded" > gpurun_out/r2x_pytest_tma.log 2>&1
echo "rc=$?" >> gpurun_out/r2x_pytest_tma.log
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2x_bench_$tag.json 2> gpurun_out/r2x_bench_$tag.err
}
run base 4
run tma 4 SBBF_SCATTER_TMA=1
run base_b 4
run tma_b 4 SBBF_SCATTER_TMA=1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
SBBF_SCATTER_TMA=1 timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2x_launch_tma_lookup.csv python scripts/profile_phase.py 4 lookup > /dev/null 2>&1
SBBF_SCATTER_TMA=1 timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2x_launch_tma_insert.csv python scripts/profile_phase.py 4 insert > /dev/null 2>&1
