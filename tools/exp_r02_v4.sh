#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
python tools/variant_time.py c3_rmat20 per_edge default $V/libgdgpu_nt512.so > gpurun_out/var_nt_pe.log 2>&1
python tools/variant_time.py c3_rmat20 global default $V/libgdgpu_nt512.so > gpurun_out/var_nt_gl.log 2>&1
python tools/variant_time.py c5_chung_lu_4m per_edge GD_C4_TILES=2 > gpurun_out/var_c5pe_tiles.log 2>&1
