# per-kernel device time + DRAM bytes of one census (ncu launch list), C3 both
# modes and C5 per-edge; summarised into profiles/ncu_summary.json by ncu_sum.py
R=${1:-r01}
for mode in per_edge global; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/${R}_c3_${mode}_dram.csv \
      python tools/profile_census.py c3_rmat20 $mode > gpurun_out/${R}_dram_${mode}.log 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${R}_c5_per_edge_dram.csv \
    python tools/profile_census.py c5_chung_lu_4m per_edge > gpurun_out/${R}_dram_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline \
    > gpurun_out/${R}_ncu_bench.log 2>&1
ls -la gpurun_out | tail -n 8
