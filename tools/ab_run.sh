for v in "" "MDHB_TC_GROUP=1" "MDHB_TC_GROUP=2" "MDHB_TC_GROUP=64"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:tf32 50 2>&1 | tail -1 | cut -c1-100
  echo "Cb $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:bf16 50 2>&1 | tail -1 | cut -c1-100
done
for v in "" "MDHB_TC_GROUP=1"; do
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 10 2>&1 | tail -1 | cut -c1-100
done
