for c in c5_chung_lu_4m c3_rmat20; do
  timeout 1200 python tools/variant_time.py $c per_edge GD_C4_FLOW_MB=128 GD_C4_FLOW_MB=256 GD_C4_FLOW_MB=960 GD_C4_FLOW_MB=1920 2>&1 | sed "s/^/$c /"
done
