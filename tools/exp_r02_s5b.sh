#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/s5b_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5b_tests.log
python tools/variant_time.py c3_rmat20 per_edge default $V/libgdgpu_norows.so $V/libgdgpu_ru2.so > gpurun_out/s5b_c3_pe.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge default $V/libgdgpu_norows.so $V/libgdgpu_ru2.so > gpurun_out/s5b_c5_pe.log 2>&1
python tools/variant_time.py c2_chung_lu per_edge default $V/libgdgpu_norows.so > gpurun_out/s5b_c2_pe.log 2>&1
