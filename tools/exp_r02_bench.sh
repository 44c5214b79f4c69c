#!/bin/bash
cd /root/repo
python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
GD_BENCH_DEBUG=1 python bench.py --steps 10 --warmup 3 --no-big --no-batch --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
