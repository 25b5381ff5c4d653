set -x
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2au_bench_$tag.json 2> gpurun_out/r2au_bench_$tag.err; }
run c64
run c32 SBBF_SEG_CHUNKS=32
run c48 SBBF_SEG_CHUNKS=48
run c96 SBBF_SEG_CHUNKS=96
run c128 SBBF_SEG_CHUNKS=128
