#!/bin/bash
cd /root/repo
for mode in per_edge; do
python tools/profile_census.py c3_rmat20 $mode > gpurun_out/prof_plain_$mode.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_c4_tiles" -s 1 -c 1 \
    -o gpurun_out/tiles_$mode python tools/profile_census.py c3_rmat20 $mode > gpurun_out/ncu_tiles_$mode.log 2>&1
done
