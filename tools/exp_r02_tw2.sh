#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "forced or default_paths or emulated or mixed or config3" > gpurun_out/tw2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/tw2_tests.log
rm -f gpurun_out/tw2_sweep.log
python tools/sweep_env.py c3_rmat20 GD_C4_TILE_LEAVES 1,0 per_edge >> gpurun_out/tw2_sweep.log 2>&1
python tools/sweep_env.py c3_rmat20 GD_C4_TILE_LEAVES 0 global >> gpurun_out/tw2_sweep.log 2>&1
python tools/sweep_env.py c3_rmat20 GD_C4_HEAVY_MIN 12288,4096,1024 per_edge >> gpurun_out/tw2_sweep.log 2>&1
python tools/sweep_env.py c3_rmat20 GD_C4_TILE 98304,81920 per_edge >> gpurun_out/tw2_sweep.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_C4_TILE_LEAVES 0 per_edge >> gpurun_out/tw2_sweep.log 2>&1
python tools/sweep_env.py c5_chung_lu_4m GD_C4_TILE_LEAVES 0 global >> gpurun_out/tw2_sweep.log 2>&1
python tools/time_c4_parts.py > gpurun_out/c4parts.log 2>&1
