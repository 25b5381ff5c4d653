# A/B on config 4: blocked round size, persistent segment grid, plain-red
# insert segments; one ncu --set full capture of the insert segment kernel.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2t_bench_$tag.json 2> gpurun_out/r2t_bench_$tag.err
}
run base
run r29 SBBF_BLOCKED_ROUND_LOG2=29
run r30 SBBF_BLOCKED_ROUND_LOG2=30
run r30p SBBF_BLOCKED_ROUND_LOG2=30 SBBF_SEG_PERSIST=1
run r28p SBBF_SEG_PERSIST=1
run nt SBBF_SEG_INS_Q=1004
run r30np SBBF_BLOCKED_ROUND_LOG2=30 SBBF_BLOCKED_PIPELINE=0
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:segment_kernel -c 1 -o gpurun_out/r2t_seg_insert python scripts/profile_phase.py 4 insert \
  > gpurun_out/r2t_seg_insert.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:chunk_scatter -c 1 -o gpurun_out/r2t_scatter_lookup python scripts/profile_phase.py 4 lookup \
  > gpurun_out/r2t_scatter_lookup.log 2>&1
