# scratch A/B of an env-selected variant (development aid): GPU tests, then
# alternating timings of the default and the variant
V=${V:-MDHB_TC_NARROW=1}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do
for v in "" "$V"; do
  echo "M tf32 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 10 2>&1 | tail -1 | cut -c1-120
  echo "M bf16 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:bf16 10 2>&1 | tail -1 | cut -c1-120
done
done
