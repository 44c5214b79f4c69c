#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python tools/variant_time.py c3_rmat20 per_edge $V/libgdgpu_tileu4.so $V/libgdgpu_tileu6.so $V/libgdgpu_tileu8.so > gpurun_out/var_u_pe.log 2>&1
python tools/variant_time.py c3_rmat20 global $V/libgdgpu_tileu4.so $V/libgdgpu_tileu6.so $V/libgdgpu_tileu8.so > gpurun_out/var_u_gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m global default $V/libgdgpu_tileu4.so $V/libgdgpu_tileu8.so > gpurun_out/var_u_c5.log 2>&1
