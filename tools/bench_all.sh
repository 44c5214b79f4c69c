# every BASELINE config through bench.py (round summaries under profiles/)
R=${1:-r01}
for c in c1_er c2_chung_lu; do
  timeout 600 python bench.py --config $c --no-batch > gpurun_out/${R}_bench_${c}_per_edge.log 2>&1
done
timeout 600 python bench.py > gpurun_out/${R}_bench_c3_rmat20_per_edge.log 2>&1
timeout 900 python bench.py --config c5_chung_lu_4m --steps 3 --warmup 3 --no-batch > gpurun_out/${R}_bench_c5_chung_lu_4m_per_edge.log 2>&1
timeout 900 python bench.py --config c5_chung_lu_4m --mode global --steps 3 --warmup 3 --no-batch --no-global > gpurun_out/${R}_bench_c5_chung_lu_4m_global.log 2>&1
for f in gpurun_out/${R}_bench_*.log; do tail -n 1 $f | cut -c1-200; done
