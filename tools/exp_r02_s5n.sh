#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/s5n_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5n_tests.log
for m in per_edge global; do
python tools/variant_time.py c3_rmat20 $m default $V/libgdgpu_nosplit.so > gpurun_out/s5n_c3_$m.log 2>&1
python tools/variant_time.py c5_chung_lu_4m $m default $V/libgdgpu_nosplit.so > gpurun_out/s5n_c5_$m.log 2>&1
done
