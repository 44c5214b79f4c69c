#!/bin/bash
# Round-2 experiment: flow-kernel slab budget (L2-resident vs DRAM-resident counters)
cd /root/repo
python -c "import __graft_entry__ as G; G.build()" > gpurun_out/build.log 2>&1 || exit 1
for mode in per_edge global; do
  python tools/sweep_env.py c3_rmat20 GD_C4_FLOW_MB 640,256,128,96,64,48,32 $mode > gpurun_out/exp_budget_$mode.log 2>&1
done
GD_C4_SETS=3 python tools/sweep_env.py c3_rmat20 GD_C4_FLOW_MB 96,64,48 per_edge > gpurun_out/exp_budget_sets3.log 2>&1
GD_C4_SETS=6 python tools/sweep_env.py c3_rmat20 GD_C4_FLOW_MB 96,64 per_edge > gpurun_out/exp_budget_sets6.log 2>&1
