#!/bin/bash
cd /root/repo
python tools/time_small.py > gpurun_out/small_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_small_census" -s 8 -c 2 \
    -o gpurun_out/small python tools/time_small.py > gpurun_out/ncu_small.log 2>&1
