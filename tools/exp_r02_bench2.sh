#!/bin/bash
cd /root/repo
python tools/census_stats.py c3_rmat20 per_edge 4 > gpurun_out/diag_c3.log 2>&1
GD_BENCH_DEBUG=1 python bench.py --steps 10 --warmup 3 --no-big --no-batch --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err
OMP_NUM_THREADS=1 python bench.py --steps 10 --warmup 3 --no-big --no-batch --no-cpu-baseline > gpurun_out/bench_omp1.log 2> gpurun_out/bench_omp1.err
