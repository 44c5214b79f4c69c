#!/bin/bash
cd /root/repo
python -m pytest tests -x -q -m gpu > gpurun_out/s5i_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5i_tests.log
for m in per_edge global; do
python tools/variant_time.py c3_rmat20 $m default > gpurun_out/s5i_c3_$m.log 2>&1
python tools/variant_time.py c5_chung_lu_4m $m default > gpurun_out/s5i_c5_$m.log 2>&1
done
python tools/variant_time.py c2_chung_lu per_edge default > gpurun_out/s5i_c2.log 2>&1
python tools/time_small.py > gpurun_out/s5i_small.log 2>&1
