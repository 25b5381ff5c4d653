set -x
mkdir -p gpurun_out
SBBF_SEG_INS_Q=1004 timeout 600 python scripts/insert_dup_probe.py 2 > gpurun_out/r2ak_nt.log 2>&1
SBBF_SEG_INS_Q=1004 SBBF_SEG_INS_PF=-2 timeout 600 python scripts/insert_dup_probe.py 2 > gpurun_out/r2ak_nt_warm.log 2>&1
