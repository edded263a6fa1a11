# scratch (development aid): GPU tests, MCC FFMA default timing and its space
timeout 1300 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do
  echo "F"; timeout 120 python tools/graph_time.py mcc_nhwc 10 2>&1 | tail -1 | cut -c1-120
done
timeout 900 python tools/space_sweep.py mcc_nhwc contraction 0 2>&1 | head -12
