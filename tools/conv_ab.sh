for v in "MDHB_TC_1SM=1" "MDHB_TC_1SM=1 MDHB_CONV_SW128=1" "MDHB_TC_1SM=1 MDHB_CONV_SW128=1 MDHB_CONV_BO=1"; do
  echo "== $v"; env $v timeout 120 python -m pytest tests/test_gpu_tc.py -x -q -k "conv or mcc" 2>&1 | tail -1
  env $v timeout 100 python tools/quick_time.py mcc_nhwc:tf32 | cut -c1-110
done
