set -x
mkdir -p gpurun_out
for pf in 0 -2; do
  SBBF_SEG_INS_PF=$pf timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aj_pf$pf.log 2>&1
done
SBBF_SEG_INS_PF=-2 SBBF_SEG_CHUNKS=128 timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aj_pf-2_c128.log 2>&1
SBBF_SEG_INS_PF=-2 SBBF_SEG_CHUNKS=32 timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2aj_pf-2_c32.log 2>&1
