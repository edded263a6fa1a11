timeout 600 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py -m gpu -q -k "not tf32 and not bf16" 2>&1 | tail -2
for v in "" "MDHB_SGEMM_NO_KLIN=1"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-100
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-100
done
