set -x
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --config 4 --extra "" --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-widened > gpurun_out/r2p_bench_$tag.json 2> gpurun_out/r2p_bench_$tag.err
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2p_launch_$tag.csv python scripts/profile_phase.py 4 lookup > /dev/null 2>&1
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2p_launchins_$tag.csv python scripts/profile_phase.py 4 insert > /dev/null 2>&1
}
run p16
run p8 SBBF_SEG_ITEM_CHUNKS=8
run p32 SBBF_SEG_ITEM_CHUNKS=32
run p4 SBBF_SEG_ITEM_CHUNKS=4
run np SBBF_SEG_PERSIST=0
