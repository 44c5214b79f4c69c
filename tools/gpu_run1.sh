timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/t_flow.log 2>&1; echo rc=$? >> gpurun_out/t_flow.log
timeout 900 python bench.py > gpurun_out/bench_flow.log 2>&1; echo rc=$? >> gpurun_out/bench_flow.log
timeout 900 python tools/sweep_env.py c5_chung_lu_4m GD_C4_MIN_CHUNK 16384 per_edge > gpurun_out/sw_flow.log 2>&1
timeout 900 python tools/sweep_env.py c5_chung_lu_4m GD_C4_MIN_CHUNK 16384 global >> gpurun_out/sw_flow.log 2>&1
