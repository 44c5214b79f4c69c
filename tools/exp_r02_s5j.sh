#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/s5j_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5j_tests.log
for m in per_edge global; do
python tools/variant_time.py c3_rmat20 $m default > gpurun_out/s5j_c3_$m.log 2>&1
python tools/variant_time.py c5_chung_lu_4m $m default > gpurun_out/s5j_c5_$m.log 2>&1
done
python tools/variant_time.py c2_chung_lu per_edge default > gpurun_out/s5j_c2.log 2>&1
