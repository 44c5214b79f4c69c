timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 600 python tools/e2e_breakdown.py c3_rmat20 > gpurun_out/e2e.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r01.log 2>&1
