# Fused sweep: is the next-slice pull worth it when it is timely (lockstep pacing, or 16 MiB slices)?
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2cs_bench_$tag.json 2> gpurun_out/r2cs_bench_$tag.err
}
run s2 4 SBBF_FUSED_SLACK=2
run s1 4 SBBF_FUSED_SLACK=1
run s1pull 4 SBBF_FUSED_SLACK=1 SBBF_FUSED_PULL=1
run m16s2 4 SBBF_SLICE_MB=16 SBBF_FUSED_SLACK=2
run m16s2pull 4 SBBF_SLICE_MB=16 SBBF_FUSED_SLACK=2 SBBF_FUSED_PULL=1
run m16s3pull 4 SBBF_SLICE_MB=16 SBBF_FUSED_SLACK=3 SBBF_FUSED_PULL=1
