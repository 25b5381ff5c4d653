# Fused lookup sweep (packed staging, shared-memory result rows): parity subset, then A/B on config 4.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "blocked or config_full or random_parity or unaligned or regions or sharded or dist" > gpurun_out/r2ca_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ca_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ca_bench_$tag.json 2> gpurun_out/r2ca_bench_$tag.err
}
run fused 4 SBBF_FIND_FUSED=1
run legacy 4 SBBF_FIND_FUSED=0
run fused_pf 4 SBBF_FIND_FUSED=1 SBBF_FUSED_PREFETCH=1
