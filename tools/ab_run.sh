# scratch A/B of an env-selected variant (development aid): parity of the
# tensor-core tests with the variant on, then alternating timings
V=${V:-MDHB_TC_WIDE=1}
env $V timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do
for v in "" "$V"; do
  echo "M tf32 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 10 2>&1 | tail -1 | cut -c1-200
  echo "M bf16 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:bf16 10 2>&1 | tail -1 | cut -c1-200
done
done
