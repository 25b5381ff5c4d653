set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2r_bench_$tag.json 2> gpurun_out/r2r_bench_$tag.err
}
run c3d 3
run c3v3 3 SBBF_SPLIT_VARIANT=3
run c3v4 3 SBBF_SPLIT_VARIANT=4
run c3v5 3 SBBF_SPLIT_VARIANT=5
bash scripts/gpu_profile_r2_traffic.sh
