# scratch A/B (development aid): FFMA default tile 128x64 vs 128x128
timeout 1300 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do
for v in "" "MDHB_PIPE_128x128=1"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-80
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-80
done
done
