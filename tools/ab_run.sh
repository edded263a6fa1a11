# scratch A/B (development aid): GPU tests, then CCSD(T) / MatMul timings
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
for v in "" "MDHB_TC_NO_RBN=1"; do
  echo "C tf32 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:tf32 50 2>&1 | tail -1 | cut -c1-110
  echo "C bf16 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:bf16 50 2>&1 | tail -1 | cut -c1-110
done
done
