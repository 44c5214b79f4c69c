#!/bin/bash
cd /root/repo
python tools/sweep_env.py c5_chung_lu_4m GD_TRI_BLOCKED 1,0 global > gpurun_out/s5t_c5.log 2>&1
python tools/sweep_env.py c3_rmat20 GD_TRI_BLOCKED 1,0 global > gpurun_out/s5t_c3.log 2>&1
