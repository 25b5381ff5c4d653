set -x
mkdir -p gpurun_out
for c in 4 6 8; do
  SBBF_UNPERM_CTAS=$c timeout 300 python bench.py --config 4 --extra "" --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2aq_bench_u$c.json 2> gpurun_out/r2aq_bench_u$c.err
done
