#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/cmp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/cmp_tests.log
python tools/variant_time.py c3_rmat20 per_edge default $V/libgdgpu_noindex.so $V/libgdgpu_nocompact.so > gpurun_out/cmp_c3_pe.log 2>&1
python tools/variant_time.py c3_rmat20 global default > gpurun_out/cmp_c3_gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge default $V/libgdgpu_noindex.so $V/libgdgpu_nocompact.so > gpurun_out/cmp_c5_pe.log 2>&1
python tools/variant_time.py c5_chung_lu_4m global default > gpurun_out/cmp_c5_gl.log 2>&1
python tools/time_c4_parts.py > gpurun_out/c4parts.log 2>&1
