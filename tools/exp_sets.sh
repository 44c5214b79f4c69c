# use-lag x slab-set sweep of the pass-C flow kernel
for c in c3_rmat20 c5_chung_lu_4m; do
  timeout 900 python tools/variant_time.py $c per_edge default "GD_C4_ULAG=2" "GD_C4_SETS=5" 2>&1 | sed "s/^/$c /"
  GD_C4_ULAG=2 timeout 900 python tools/variant_time.py $c per_edge GD_C4_SETS=5 GD_C4_SETS=6 2>&1 | sed "s/^/$c ULAG=2 /"
done
timeout 900 python tools/variant_time.py c3_rmat20 global default GD_C4_ULAG=2 2>&1 | sed "s/^/c3 global /"
