for c in c3_rmat20 c5_chung_lu_4m; do
  timeout 900 python tools/variant_time.py $c per_edge default GD_WIDE_SLOTS=1 2>&1 | sed "s/^/$c /"
done
