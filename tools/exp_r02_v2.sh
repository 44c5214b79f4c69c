#!/bin/bash
cd /root/repo
python tools/variant_time.py c5_chung_lu_4m per_edge GD_C4_TILES=1 GD_C4_TILES=2 > gpurun_out/var_c5_pe.log 2>&1
