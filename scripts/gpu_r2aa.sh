# Insert phase with vs without config 4's Zipf duplicates (defaults: TMA
# partition, no lookup pipeline); the same with the LSU partition.
set -x
mkdir -p gpurun_out
timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aa_dup.log 2>&1
SBBF_SCATTER_TMA=0 timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aa_dup_lsu.log 2>&1
SBBF_SEG_INS_Q=6008 timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aa_dup_lean8.log 2>&1
SBBF_SEG_INS_Q=1004 timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aa_dup_notest.log 2>&1
