#!/bin/bash
cd /root/repo
python -m pytest tests -x -q -m gpu -k "batch or feature or analytics or small or edge_cases or workloads" > gpurun_out/s5q_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5q_tests.log
GD_HOST_PROFILE=1 python tools/time_c4_parts.py > gpurun_out/s5q_c4.log 2>&1
python tools/time_small.py > gpurun_out/s5q_small.log 2>&1
