# C5 bench lines + a source-level ncu capture of the pass-C flow kernel (C3 per-edge)
set -x
timeout 900 python bench.py --config c5_chung_lu_4m --steps 3 --warmup 3 --no-batch > gpurun_out/bench_c5_per_edge.log 2>&1
timeout 600 python bench.py --config c5_chung_lu_4m --mode global --steps 3 --warmup 3 --no-batch --no-global > gpurun_out/bench_c5_global.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_c4_flow -s 1 -c 1 \
    -o gpurun_out/r01_flow_src python tools/profile_census.py c3_rmat20 per_edge \
    > gpurun_out/r01_flow_src.log 2>&1
ls -la gpurun_out
