timeout 900 python tools/time_selection.py c2_chung_lu > gpurun_out/time_sel.log 2>&1
timeout 900 python tools/time_selection.py c3_rmat20 >> gpurun_out/time_sel.log 2>&1
