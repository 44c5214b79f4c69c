# Round profile captures (run on the GPU box via gpurun; one GPU, never
# multi-rank).  Outputs land in gpurun_out/ (keep them < 64 MiB) and are
# summarised into profiles/ by tools/ncu_sum.py and tools/ncu_full_json.py.
R=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 1 \
    > gpurun_out/${R}_ncu_bench.log 2>&1
for mode in per_edge global; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/${R}_c3_${mode}_dram.csv \
      python tools/profile_census.py c3_rmat20 $mode > gpurun_out/${R}_dram_${mode}.log 2>&1
done
# full sets of every counting kernel of both censuses -> JSON (report deleted)
ncu --set full --clock-control none \
    -k regex:"k_c4_flow|k_tri_frames|k_trisum_frames|k_c4_frames_smem" -c 60 \
    -o /tmp/${R}_full_c3 python tools/profile_census.py c3_rmat20 per_edge \
    > gpurun_out/${R}_full.log 2>&1
python tools/ncu_full_json.py /tmp/${R}_full_c3.ncu-rep > gpurun_out/${R}_ncu_full_c3_per_edge.json
# source-level capture of the dominant kernel only
ncu --set full --clock-control none --import-source on -k regex:k_c4_flow -s 1 -c 1 \
    -o gpurun_out/${R}_flow_src python tools/profile_census.py c3_rmat20 per_edge \
    > gpurun_out/${R}_flow_src.log 2>&1
du -sh gpurun_out
echo done
