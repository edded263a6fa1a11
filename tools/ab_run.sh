# scratch (development aid): GPU tests + FFMA defaults timing
timeout 1300 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do
  echo "C"; timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-100
  echo "M"; timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-100
  echo "F"; timeout 120 python tools/graph_time.py mcc_nhwc 10 2>&1 | tail -1 | cut -c1-100
done
