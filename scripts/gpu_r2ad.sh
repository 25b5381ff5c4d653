# A/B: bulk L2 prefetch of the slice k steps ahead in the insert sweep
set -x
mkdir -p gpurun_out
for pf in 0 1 2 -1 3; do
  SBBF_SEG_INS_PF=$pf timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2ad_pf$pf.log 2>&1
done
for pf in 0 1 2; do
  SBBF_SEG_INS_PF=$pf SBBF_SLICE_MB=16 timeout 600 python scripts/insert_dup_probe.py 3 > gpurun_out/r2ad_pf${pf}_s16.log 2>&1
done
