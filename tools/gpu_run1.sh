timeout 900 python -m pytest tests/test_gpu_edgelist.py -x -q -s > gpurun_out/t_parse.log 2>&1; echo rc=$? >> gpurun_out/t_parse.log
timeout 900 python tools/time_parse.py c3_rmat20 > gpurun_out/time_parse.log 2>&1
