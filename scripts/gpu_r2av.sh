set -x
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2av_bench_$tag.json 2> gpurun_out/r2av_bench_$tag.err; }
run pf0
run pf128 SBBF_SEG_L2PF=128
run pf256 SBBF_SEG_L2PF=256
