# scratch A/B (development aid): 192-column FFMA instances on CCSD(T)
for v in "MDHB_SGEMM_192=64" "MDHB_SGEMM_192=128"; do
  env $v timeout 900 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py -m gpu -q -x -k "ccsdt" 2>&1 | tail -1
done
for i in 1 2; do
for v in "" "MDHB_SGEMM_192=64" "MDHB_SGEMM_192=128"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-100
done
done
