# scratch A/B (development aid): 24-deep k-tiles on the 128x64 FFMA instance
MDHB_SGEMM_BK24=1 timeout 600 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py -m gpu -q -x -k ccsdt 2>&1 | tail -1
for i in 1 2; do
for v in "" "MDHB_SGEMM_BK24=1"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-100
done
done
