#!/bin/bash
cd /root/repo
V=paper_1506_04322_b200/_variants
for m in per_edge global; do
python tools/variant_time.py c3_rmat20 $m default $V/libgdgpu_pm64.so $V/libgdgpu_pm256.so $V/libgdgpu_pm512.so > gpurun_out/s5g_c3_$m.log 2>&1
python tools/variant_time.py c5_chung_lu_4m $m default $V/libgdgpu_pm64.so $V/libgdgpu_pm256.so $V/libgdgpu_pm512.so > gpurun_out/s5g_c5_$m.log 2>&1
done
