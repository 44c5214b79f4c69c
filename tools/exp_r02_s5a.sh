#!/bin/bash
cd /root/repo
python -m pytest tests -m gpu -x -q > gpurun_out/s5a_gputests.log 2>&1
echo "rc=$?" >> gpurun_out/s5a_gputests.log
python tools/e2e_breakdown.py c3_rmat20 > gpurun_out/s5a_e2e_c3.log 2>&1
python bench.py > gpurun_out/s5a_bench.log 2>&1
echo "rc=$?" >> gpurun_out/s5a_bench.log
