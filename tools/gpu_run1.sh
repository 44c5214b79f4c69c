timeout 900 python tools/time_derive.py c3_rmat20 > gpurun_out/time_derive.log 2>&1
