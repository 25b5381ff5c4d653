# ncu --set full of one fused lookup sweep (6 CTAs/SM, paced) on config 4.
set -x
mkdir -p gpurun_out
SBBF_FUSED_VARIANT=3 SBBF_FUSED_SLACK=2 ncu --set full --import-source on --clock-control none -k regex:"sweep_find" -c 1 -o gpurun_out/r2cj_sweep_find -f python scripts/profile_blocked.py 4 find 3 1 > gpurun_out/r2cj_ncu.log 2>&1
