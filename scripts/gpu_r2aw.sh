set -x
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2aw_bench_$tag.json 2> gpurun_out/r2aw_bench_$tag.err; }
run new
run old SBBF_SEG_CHUNKS=64
run new2
