#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -k "forced or config3 or small_graph" > gpurun_out/v1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/v1_tests.log
bash tools/exp_r02_variants.sh
