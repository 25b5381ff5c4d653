# A/B: flat-sequence lookup sweep (new defaults: TMA partition + unpermute).
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ab_bench_$tag.json 2> gpurun_out/r2ab_bench_$tag.err
}
run def 4
run flat 4 SBBF_SEG_FLAT=1
run flat32 4 SBBF_SEG_FLAT=1 SBBF_SEG_CHUNKS=32
run flat128 4 SBBF_SEG_FLAT=1 SBBF_SEG_CHUNKS=128
SBBF_SEG_FLAT=1 timeout 900 python -m pytest tests -m gpu -q -x -k "blocked or config_full or random_parity or golden_filters" > gpurun_out/r2ab_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ab_pytest.log
