#!/bin/bash
# SASS listings of the census kernels that bound the configs (evidence for
# the kernel design: shared-memory atomics ATOMS / LDS in the tile and small
# kernels, REDG slot updates, no local-memory spills in the hot loops).
# Usage: tools/dump_sass.sh [outdir]   (builds a cubin of gd_count.cu)
OUT=${1:-profiles/r02_sass}
mkdir -p $OUT
ROOT=$(cd $(dirname $0)/.. && pwd)
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
  -I$ROOT/include -cubin -o /tmp/gd_count_sass.cubin $ROOT/paper_1506_04322_b200/csrc/gd_count.cu
for pat in "k_c4_tilesILi1024EjiE" "k_tri_framesILi512ELb0ELb0E" "k_trisum_framesILi512ELb0EjjE" \
           "k_finalize_singleILi256E" "k_c4_flowILi512ELi4ELi1ELi2EjE" "k_small_censusILi256ELb1ELb0E" \
           "k_small_censusILi128ELb0ELb1E" "k_c4_frames_smemILi1024ELb1EjE"; do
  fn=$(cuobjdump -elf /tmp/gd_count_sass.cubin | grep -o "\.text\.[^ ]*$pat[^ ]*" | head -1 | sed 's/^\.text\.//')
  [ -z "$fn" ] && { echo "missing $pat"; continue; }
  name=$(echo $pat | sed 's/ILi/_/; s/E.*//')
  cuobjdump -sass -fun "$fn" /tmp/gd_count_sass.cubin > $OUT/$name.sass
  printf "%-34s %6d instr  ATOMS %4d  LDS %4d  REDG/RED %4d  ATOMG %3d  LDG %4d  STL/LDL %d\n" $name \
    $(grep -c "^ */\*[0-9a-f]*\*/" $OUT/$name.sass) $(grep -c "ATOMS" $OUT/$name.sass) \
    $(grep -c " LDS" $OUT/$name.sass) $(grep -c " RED" $OUT/$name.sass) $(grep -c "ATOMG" $OUT/$name.sass) \
    $(grep -c " LDG" $OUT/$name.sass) $(grep -c "STL\|LDL" $OUT/$name.sass)
done
