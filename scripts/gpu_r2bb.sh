# A/B: insert sweep with the shared-memory dedup table vs test-before-set;
# config 3 lookups with 2/3/4 compacted range passes. Parity of both first.
set -x
mkdir -p gpurun_out
SBBF_SEG_DEDUP=1 timeout 900 python -m pytest tests -m gpu -q -x -k "blocked or config_full or golden_filters or random_parity or config5" > gpurun_out/r2bb_pytest_dedup.log 2>&1; echo rc=$? >> gpurun_out/r2bb_pytest_dedup.log
for P in 3 4; do
SBBF_SPLIT_PASSES=$P timeout 900 python -m pytest tests -m gpu -q -x -k "config_full or range_split or random_parity" > gpurun_out/r2bb_pytest_p$P.log 2>&1; echo rc=$? >> gpurun_out/r2bb_pytest_p$P.log
done
t() { tag=$1; shift; env "$@" timeout 300 python scripts/insert_dup_probe.py 3 > gpurun_out/r2bb_ins_$tag.log 2>&1; }
t q2
t q4 SBBF_SEG_INS_Q=4
t q2d SBBF_SEG_DEDUP=1
t q4d SBBF_SEG_DEDUP=1 SBBF_SEG_INS_Q=4
t q2d32 SBBF_SEG_DEDUP=1 SBBF_SEG_CHUNKS=32
t q4d32 SBBF_SEG_DEDUP=1 SBBF_SEG_INS_Q=4 SBBF_SEG_CHUNKS=32
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 3 --extra "" --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2bb_c3_$tag.json 2> gpurun_out/r2bb_c3_$tag.err; }
b p2
b p3 SBBF_SPLIT_PASSES=3
b p4 SBBF_SPLIT_PASSES=4
