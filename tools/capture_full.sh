# bench launch list + full-set captures of the census kernels (C3 per-edge)
R=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline \
    > gpurun_out/${R}_ncu_bench.log 2>&1
ncu --set full --clock-control none \
    -k regex:"k_c4_flow|k_tri_frames|k_trisum_frames|k_c4_frames_smem|k_finalize" -c 40 \
    -o /tmp/${R}_full_c3 python tools/profile_census.py c3_rmat20 per_edge \
    > gpurun_out/${R}_full.log 2>&1
python tools/ncu_full_json.py /tmp/${R}_full_c3.ncu-rep > gpurun_out/${R}_ncu_full_c3_per_edge.json
tail -n 3 gpurun_out/${R}_full.log
