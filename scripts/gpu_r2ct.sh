# Timing diagnostics of the fused sweep (wrong answers by construction, never shipped):
# diagwin = every probe inside 8 KB of its slice; diagnokeys = slots synthesised (no slot stream); both.
set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ct_bench_$tag.json 2> gpurun_out/r2ct_bench_$tag.err
}
run base
run diagwin SBBF_LIB=diagwin
run diagnokeys SBBF_LIB=diagnokeys
run diagboth SBBF_LIB=diagboth
run diagboth_free SBBF_LIB=diagboth SBBF_FUSED_SLACK=0
run diagboth_v1 SBBF_LIB=diagboth SBBF_FUSED_VARIANT=1
