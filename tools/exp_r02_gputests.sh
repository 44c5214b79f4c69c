#!/bin/bash
cd /root/repo
python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
