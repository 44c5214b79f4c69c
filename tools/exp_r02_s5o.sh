#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "forced" > gpurun_out/s5o_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s5o_tests.log
python tools/sweep_env.py c3_rmat20 GD_C4_PIECE_MIN 192,256,384 per_edge > gpurun_out/s5o_c3.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_C4_PIECE_MIN 96,128,192,256 per_edge > gpurun_out/s5o_c5.log 2>&1
