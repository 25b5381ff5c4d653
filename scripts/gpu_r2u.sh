# A/B on config 4 lookups: co-resident partition (side stream, 1 CTA/SM) and
# persistent probe grid sized to leave it room; 3 scratch buffers.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2u_bench_$tag.json 2> gpurun_out/r2u_bench_$tag.err
}
run base
run o1 SBBF_PART_PER_SM=1 SBBF_PIPE_BUFS=3 SBBF_SEG_PERSIST=2 SBBF_SEG_PERSIST_CTAS=4
run o2 SBBF_PART_PER_SM=1 SBBF_PIPE_BUFS=3 SBBF_SEG_PERSIST=2 SBBF_SEG_PERSIST_CTAS=2 SBBF_SEG_LOOK_Q=2
run o3 SBBF_PART_PER_SM=1 SBBF_PIPE_BUFS=3
run o4 SBBF_PIPE_BUFS=3 SBBF_SEG_PERSIST=2 SBBF_SEG_PERSIST_CTAS=4
run o5 SBBF_PART_PER_SM=1 SBBF_PIPE_BUFS=3 SBBF_SEG_PERSIST=2 SBBF_SEG_PERSIST_CTAS=3
run o6 SBBF_PART_PER_SM=1 SBBF_PIPE_BUFS=2 SBBF_SEG_PERSIST=2 SBBF_SEG_PERSIST_CTAS=4
