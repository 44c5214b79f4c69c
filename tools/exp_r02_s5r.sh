#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/s5r_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5r_tests.log
for m in per_edge global; do
python tools/sweep_env.py c3_rmat20 GD_C4_JOB_ORDER 0,1,2 $m > gpurun_out/s5r_c3_$m.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_C4_JOB_ORDER 0,1,2 $m > gpurun_out/s5r_c5_$m.log 2>&1
done
