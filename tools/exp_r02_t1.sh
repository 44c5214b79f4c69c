#!/bin/bash
# tile fast path / 32-bit slot index variants
cd /root/repo
V=paper_1506_04322_b200/_variants
timeout 900 python -m pytest tests -m gpu -x -q -k "forced or config3 or tile or edge_cases" > gpurun_out/t1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/t1_tests.log
python tools/variant_time.py c3_rmat20 per_edge default GD_TILE_IDX32=0 $V/libgdgpu_nofast.so $V/libgdgpu_u2.so $V/libgdgpu_u6.so $V/libgdgpu_u8.so > gpurun_out/t1_c3pe.log 2>&1
python tools/variant_time.py c3_rmat20 global default GD_TILE_IDX32=0 $V/libgdgpu_nofast.so $V/libgdgpu_u2.so $V/libgdgpu_u8.so > gpurun_out/t1_c3gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m global default $V/libgdgpu_nofast.so $V/libgdgpu_u8.so > gpurun_out/t1_c5gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge default $V/libgdgpu_nofast.so $V/libgdgpu_u8.so > gpurun_out/t1_c5pe.log 2>&1
python tools/time_c4_parts.py > gpurun_out/t1_c4parts.log 2>&1
