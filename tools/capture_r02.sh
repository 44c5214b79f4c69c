#!/bin/bash
# Round-2 evidence: per-kernel DRAM of one census (C3, C5 both modes), full-set
# metrics of the dominant kernels, and the bench launch list.  Every ncu run
# follows a plain run of the same command that exited 0.
cd "$(dirname "$0")/.."
R=r02
set -x
for cfg in c3_rmat20 c5_chung_lu_4m; do
  for mode in per_edge global; do
    python tools/profile_census.py $cfg $mode > gpurun_out/${R}_plain_${cfg}_${mode}.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/${R}_${cfg}_${mode}_dram.csv \
        python tools/profile_census.py $cfg $mode > gpurun_out/${R}_dram_${cfg}_${mode}.log 2>&1
  done
done
python tools/profile_census.py c3_rmat20 per_edge > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_c4_tiles|k_tri_frames|k_trisum_frames|k_c4_frames_smem|k_finalize" -c 40 \
    -o /tmp/${R}_full_c3 python tools/profile_census.py c3_rmat20 per_edge \
    > gpurun_out/${R}_full_c3.log 2>&1
python tools/ncu_full_json.py /tmp/${R}_full_c3.ncu-rep > gpurun_out/${R}_ncu_full_c3_per_edge.json
python tools/ncu_source_top.py /tmp/${R}_full_c3.ncu-rep 12 > gpurun_out/${R}_source_c3_per_edge.json
python tools/profile_census.py c5_chung_lu_4m per_edge > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_c4_tiles|k_tri_frames<1024" -c 4 \
    -o /tmp/${R}_full_c5 python tools/profile_census.py c5_chung_lu_4m per_edge \
    > gpurun_out/${R}_full_c5.log 2>&1
python tools/ncu_full_json.py /tmp/${R}_full_c5.ncu-rep > gpurun_out/${R}_ncu_full_c5_per_edge.json
python tools/ncu_source_top.py /tmp/${R}_full_c5.ncu-rep 12 > gpurun_out/${R}_source_c5_per_edge.json
python tools/time_small.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_small_census" -s 6 -c 2 \
    -o /tmp/${R}_full_small python tools/time_small.py > gpurun_out/${R}_full_small.log 2>&1
python tools/ncu_full_json.py /tmp/${R}_full_small.ncu-rep > gpurun_out/${R}_ncu_full_small.json
python tools/ncu_source_top.py /tmp/${R}_full_small.ncu-rep 12 > gpurun_out/${R}_source_small.json
python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline --no-big > gpurun_out/${R}_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-batch \
    --no-cpu-baseline --no-big > gpurun_out/${R}_ncu_bench.log 2>&1
du -sh gpurun_out; ls -la gpurun_out | tail -n 30
