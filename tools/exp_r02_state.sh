#!/bin/bash
# Round-2 re-entry: full GPU suite, smoke, default bench line.
cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "rc=$?" >> gpurun_out/bench.err
