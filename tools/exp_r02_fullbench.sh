#!/bin/bash
cd /root/repo
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
echo "rc=$?" >> gpurun_out/bench_full.err
for cfg in c1_er c2_chung_lu; do
  python bench.py --config $cfg --no-big --no-batch > gpurun_out/bench_$cfg.log 2>> gpurun_out/bench_full.err
done
python bench.py --config c3_rmat20 --mode global --no-big --no-batch > gpurun_out/bench_c3_global.log 2>> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.log 2>> gpurun_out/bench_full.err
