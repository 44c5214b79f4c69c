#!/bin/bash
cd /root/repo
python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
for mode in per_edge global; do
  python tools/sweep_env.py c3_rmat20 GD_C4_TILES 1 $mode > gpurun_out/pol_c3_$mode.log 2>&1
done
