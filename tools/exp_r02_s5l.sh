#!/bin/bash
cd /root/repo
python -m pytest tests -x -q -m gpu > gpurun_out/s5l_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5l_tests.log
python tools/e2e_breakdown.py c3_rmat20 > gpurun_out/s5l_e2e_c3.log 2>&1
python bench.py > gpurun_out/s5l_bench.log 2>&1
echo "rc=$?" >> gpurun_out/s5l_bench.log
