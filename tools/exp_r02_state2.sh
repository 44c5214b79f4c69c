#!/bin/bash
cd /root/repo
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
echo "rc=$?" >> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.log 2>> gpurun_out/bench_full.err
