# scratch A/B of an env-selected variant (development aid): MCC GPU tests,
# then alternating timings of the default and the variant
V=${V:-MDHB_FCONV_NOTAIL=1}
timeout 900 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py tests/test_gpu_tc.py -m gpu -q -x -k "mcc or conv" 2>&1 | tail -3
for i in 1 2 3; do
for v in "" "$V"; do
  echo "F $v"; env $v timeout 120 python tools/graph_time.py mcc_nhwc 10 2>&1 | tail -1 | cut -c1-100
done
done
