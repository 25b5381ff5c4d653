set -x
mkdir -p gpurun_out
t() { tag=$1; shift; env "$@" timeout 300 python scripts/insert_dup_probe.py 3 > gpurun_out/r2ax_$tag.log 2>&1; }
t q4c32
t q2c16 SBBF_SEG_INS_Q=2 SBBF_SEG_CHUNKS=16
t q2c32 SBBF_SEG_INS_Q=2 SBBF_SEG_CHUNKS=32
t q8c64 SBBF_SEG_INS_Q=8 SBBF_SEG_CHUNKS=64
t q4c64 SBBF_SEG_CHUNKS=64
