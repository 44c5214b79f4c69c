timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "forced or dense or small" > gpurun_out/t_flow.log 2>&1; echo rc=$? >> gpurun_out/t_flow.log
timeout 900 python tools/sweep_env.py c3_rmat20 GD_TRI_SPLIT 1,1 per_edge > gpurun_out/sw_flow.log 2>&1
timeout 900 python tools/sweep_env.py c3_rmat20 GD_TRI_SPLIT 1 global >> gpurun_out/sw_flow.log 2>&1
timeout 900 python tools/sweep_env.py c5_chung_lu_4m GD_TRI_SPLIT 1 global >> gpurun_out/sw_flow.log 2>&1
