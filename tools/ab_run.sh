# scratch A/B (development aid): partial last k-tile in the FFMA template
timeout 900 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py tests/test_gpu_tuner_space.py tests/test_gpu_tuner.py -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do
for v in "" "MDHB_SGEMM_NO_KTAIL=1"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-100
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-100
done
done
