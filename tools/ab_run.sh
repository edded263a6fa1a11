# scratch A/B (development aid): default vs the saved baseline library (libmdh_b200_alt.so)
ALT=$PWD/paper_2405_05118_b200/libmdh_b200_alt.so
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py -m gpu -q -x -k "ccsdt or tail" 2>&1 | tail -1
for i in 1 2; do
for v in "" "MDHB_LIB=$ALT"; do
  echo "C tf32 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:tf32 50 2>&1 | tail -1 | cut -c1-70
  echo "C bf16 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:bf16 50 2>&1 | tail -1 | cut -c1-70
done
done
