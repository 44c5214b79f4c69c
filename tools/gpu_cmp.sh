#!/bin/bash
# Parity subset + phase timings of the default library against variant builds
# (tools/build_variant.py): bash tools/gpu_cmp.sh name1 name2 ...
cd "$(dirname "$0")/.."
V=paper_1506_04322_b200/_variants
libs="default"; for n in "$@"; do libs="$libs $V/libgdgpu_$n.so"; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu -k "not config5" > gpurun_out/cmp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/cmp_tests.log
for m in per_edge global; do
python tools/variant_time.py c3_rmat20 $m $libs > gpurun_out/cmp_c3_$m.log 2>&1
python tools/variant_time.py c5_chung_lu_4m $m $libs > gpurun_out/cmp_c5_$m.log 2>&1
done
