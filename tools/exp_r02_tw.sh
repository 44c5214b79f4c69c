#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "forced or default_paths or emulated or mixed or config3" > gpurun_out/tw_tests.log 2>&1
echo "rc=$?" >> gpurun_out/tw_tests.log
for b in 16 2; do
python tools/sweep_env.py c3_rmat20 GD_C4_TILE_BITS $b per_edge >> gpurun_out/tw_sweep.log 2>&1
python tools/sweep_env.py c3_rmat20 GD_C4_TILE_BITS $b global >> gpurun_out/tw_sweep.log 2>&1
done
python tools/sweep_env.py c5_chung_lu_4m GD_C4_TILE_BITS 16,2 per_edge >> gpurun_out/tw_sweep.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_C4_TILE_BITS 16,2 global >> gpurun_out/tw_sweep.log 2>&1
