#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/s5d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5d_tests.log
python tools/variant_time.py c3_rmat20 per_edge default $V/libgdgpu_nogrouped.so $V/libgdgpu_ru8.so $V/libgdgpu_k16.so $V/libgdgpu_k64.so > gpurun_out/s5d_c3_pe.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge default $V/libgdgpu_nogrouped.so $V/libgdgpu_ru8.so $V/libgdgpu_k16.so $V/libgdgpu_k64.so > gpurun_out/s5d_c5_pe.log 2>&1
