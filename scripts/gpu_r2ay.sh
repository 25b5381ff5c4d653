set -x
mkdir -p gpurun_out
t() { tag=$1; shift; env "$@" timeout 300 python scripts/insert_dup_probe.py 3 > gpurun_out/r2ay_$tag.log 2>&1; }
t q2c16 SBBF_SEG_INS_Q=2 SBBF_SEG_CHUNKS=16
t q1c8 SBBF_SEG_INS_Q=1 SBBF_SEG_CHUNKS=8
t q1c16 SBBF_SEG_INS_Q=1 SBBF_SEG_CHUNKS=16
t q2c24 SBBF_SEG_INS_Q=2 SBBF_SEG_CHUNKS=48
