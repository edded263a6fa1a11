# scratch A/B (development aid): FFMA contraction parity, then timings
python tools/describe_probe.py 2>&1 | cut -c1-300
timeout 900 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
for v in "" "MDHB_SGEMM_NO_BULK=1"; do
  echo "C $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-100
done
done
