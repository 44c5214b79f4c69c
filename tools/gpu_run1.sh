timeout 900 python tools/sweep_env.py c5_chung_lu_4m GD_TRI_GM_NT 512,1024 global > gpurun_out/sw_flow.log 2>&1
timeout 900 python tools/sweep_env.py c5_chung_lu_4m GD_TRI_GM_NT 512,1024 per_edge >> gpurun_out/sw_flow.log 2>&1
