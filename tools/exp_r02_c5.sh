#!/bin/bash
cd /root/repo
for mode in per_edge global; do
  python tools/sweep_env.py c5_chung_lu_4m GD_C4_TILES 1,0 $mode > gpurun_out/tiles_c5_$mode.log 2>&1
done
