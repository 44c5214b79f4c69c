#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python tools/variant_time.py c3_rmat20 per_edge default $V/libgdgpu_nopf.so > gpurun_out/var_pf_c3pe.log 2>&1
python tools/variant_time.py c3_rmat20 global default $V/libgdgpu_nopf.so > gpurun_out/var_pf_c3gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m global default $V/libgdgpu_nopf.so > gpurun_out/var_pf_c5gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge default $V/libgdgpu_nopf.so > gpurun_out/var_pf_c5pe.log 2>&1
