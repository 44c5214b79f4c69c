#!/bin/bash
# Full GPU check: parity suite, e2e breakdown and the default bench line.
cd "$(dirname "$0")/.."
python -m pytest tests -x -q -m gpu > gpurun_out/chk_tests.log 2>&1
echo "rc=$?" >> gpurun_out/chk_tests.log
python tools/e2e_breakdown.py c3_rmat20 > gpurun_out/chk_e2e_c3.log 2>&1
python bench.py > gpurun_out/chk_bench.log 2>&1
echo "rc=$?" >> gpurun_out/chk_bench.log
GD_D2H_OVERLAP=0 python bench.py --no-batch --no-cpu-baseline --no-global --no-big > gpurun_out/chk_bench_nooverlap.log 2>&1
