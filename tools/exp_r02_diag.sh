#!/bin/bash
cd /root/repo
GD_HIT_WS=1 python tools/census_stats.py c5_chung_lu_4m per_edge 3 > gpurun_out/diag_c5_ws.log 2>&1
GD_HIT_CAP=9000000000 python tools/census_stats.py c5_chung_lu_4m per_edge 3 > gpurun_out/diag_c5_cap.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_HIT_WS 0,1 per_edge > gpurun_out/diag_c5_sweep.log 2>&1
