# Fused lookup sweep with CTA-level slice pacing and next-slice bulk prefetch: A/B on config 4.
set -x
mkdir -p gpurun_out
run() { # tag config env...
  tag=$1; cfg=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $cfg --extra "" --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2ce_bench_$tag.json 2> gpurun_out/r2ce_bench_$tag.err
}
for v in 2 3; do
 for sl in 1 2; do
  for pf in 0 1; do
   run v${v}s${sl}p${pf} 4 SBBF_FUSED_VARIANT=$v SBBF_FUSED_SLACK=$sl SBBF_FUSED_PREFETCH=$pf
  done
 done
done
run v3s0 4 SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=0
