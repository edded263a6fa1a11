ALT=$PWD/paper_2405_05118_b200/libmdh_b200_alt.so
for i in 1 2; do
for v in "" "MDHB_LIB=$ALT"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-60
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-60
  echo "F $v"; env $v timeout 120 python tools/graph_time.py mcc_nhwc 3 2>&1 | tail -1 | cut -c1-60
done
done
