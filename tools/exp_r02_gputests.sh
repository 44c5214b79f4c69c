#!/bin/bash
cd /root/repo
python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
python tools/time_small.py > gpurun_out/small.log 2>&1
python tools/time_c4_parts.py > gpurun_out/c4parts.log 2>&1
