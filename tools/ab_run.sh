# scratch A/B (development aid): FFMA conv parity, then default vs the saved
# baseline library (libmdh_b200_alt.so)
ALT=$PWD/paper_2405_05118_b200/libmdh_b200_alt.so
timeout 900 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_fullsize.py tests/test_gpu_tc.py -m gpu -q -x -k "mcc or conv" 2>&1 | tail -2
for i in 1 2; do
for v in "" "MDHB_LIB=$ALT"; do
  echo "F $v"; env $v timeout 120 python tools/graph_time.py mcc_nhwc 10 2>&1 | tail -1 | cut -c1-80
done
done
