#!/bin/bash
cd /root/repo
GD_HOST_PROFILE=1 python tools/time_c4_parts.py > gpurun_out/s5p_c4.log 2>&1
python tools/time_small.py > gpurun_out/s5p_small.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5p_launches.csv python tools/time_c4_parts.py > /dev/null 2>&1
