#!/bin/bash
cd /root/repo
python tools/sweep_env.py c3_rmat20 GD_C4_TOP_NT 1024,512 per_edge > gpurun_out/s5u_top.log 2>&1
python tools/sweep_env.py c3_rmat20 GD_C4_MID_NT 1024,512 per_edge > gpurun_out/s5u_mid.log 2>&1
