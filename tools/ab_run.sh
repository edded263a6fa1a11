# scratch A/B (development aid): wide CTA-pair TF32 GEMM, K-major B copy vs MN-major B
MDHB_TC_NO_TRANSPOSE=1 MDHB_TC_WIDE_MN=1 timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py -m gpu -q -x -k "matmul" 2>&1 | tail -1
for i in 1 2; do
for v in "" "MDHB_TC_NO_TRANSPOSE=1 MDHB_TC_WIDE_MN=1" "MDHB_TC_NO_TRANSPOSE=1"; do
  echo "M tf32 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 10 2>&1 | tail -1 | cut -c1-110
done
done
