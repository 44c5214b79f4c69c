#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python tools/variant_time.py c3_rmat20 per_edge default $V/libgdgpu_bsearch.so $V/libgdgpu_claims2.so $V/libgdgpu_claims1.so > gpurun_out/var_c3_pe.log 2>&1
python tools/variant_time.py c3_rmat20 global default $V/libgdgpu_claims2.so $V/libgdgpu_claims1.so > gpurun_out/var_c3_gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge default $V/libgdgpu_claims2.so $V/libgdgpu_claims1.so > gpurun_out/var_c5_pe.log 2>&1
