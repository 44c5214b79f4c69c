#!/bin/bash
# Round-2: x-tiled shared-memory heavy-frame kernel, correctness then timing
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -k "forced or default_paths or config1 or config2" > gpurun_out/tiles_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tiles_tests.log
for mode in per_edge global; do
  python tools/sweep_env.py c3_rmat20 GD_C4_TILES 0,1 $mode > gpurun_out/tiles_c3_$mode.log 2>&1
done
python tools/sweep_env.py c3_rmat20 GD_C4_TILE 90112,65536,49152 per_edge > gpurun_out/tiles_c3_T.log 2>&1
python tools/sweep_env.py c2_chung_lu GD_C4_TILES 0,1 per_edge > gpurun_out/tiles_c2.log 2>&1
