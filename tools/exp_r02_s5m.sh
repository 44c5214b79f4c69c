#!/bin/bash
cd /root/repo
python tools/sweep_env.py c3_rmat20 GD_C4_HEAVY_MIN 2048,4096,8192,12288,24576 per_edge > gpurun_out/s5m_c3.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_C4_HEAVY_MIN 4096,12288,24576 per_edge > gpurun_out/s5m_c5.log 2>&1
