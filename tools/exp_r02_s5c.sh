#!/bin/bash
cd /root/repo
python tools/profile_census.py c3_rmat20 per_edge > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_tri_frames|k_trisum_frames" -c 11 \
    -o /tmp/s5c_tri python tools/profile_census.py c3_rmat20 per_edge > gpurun_out/s5c_full.log 2>&1
python tools/ncu_full_json.py /tmp/s5c_tri.ncu-rep > gpurun_out/s5c_ncu_tri.json
python tools/ncu_source_top.py /tmp/s5c_tri.ncu-rep 30 > gpurun_out/s5c_source_tri.json
