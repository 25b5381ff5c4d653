set -x
mkdir -p gpurun_out
SBBF_INSERT_TILES=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:tile_scatter -c 1 -o gpurun_out/r2al_tile_scatter python scripts/profile_phase.py 4 insert > gpurun_out/r2al_ts.log 2>&1
SBBF_INSERT_TILES=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:tile_apply -c 1 -o gpurun_out/r2al_tile_apply python scripts/profile_phase.py 4 insert > gpurun_out/r2al_ta.log 2>&1
