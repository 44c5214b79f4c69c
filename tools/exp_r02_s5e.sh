#!/bin/bash
cd /root/repo
python tools/profile_census.py c3_rmat20 per_edge > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_c4_tiles" -c 1 \
    -o /tmp/s5e_tiles python tools/profile_census.py c3_rmat20 per_edge > gpurun_out/s5e_full.log 2>&1
python tools/ncu_full_json.py /tmp/s5e_tiles.ncu-rep > gpurun_out/s5e_ncu_tiles.json
python tools/ncu_source_top.py /tmp/s5e_tiles.ncu-rep 45 > gpurun_out/s5e_source_tiles.json
ncu -i /tmp/s5e_tiles.ncu-rep --page details --csv > gpurun_out/s5e_details.csv 2>&1
