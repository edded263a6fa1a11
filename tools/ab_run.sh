for v in "MDHB_SKINNY_NW=64" "MDHB_SKINNY_NW=128" "MDHB_SKINNY_NW=128 MDHB_SKINNY_CS=16"; do
  echo "T $v"; env $v timeout 300 python -m pytest tests/test_gpu_contraction.py -m gpu -q -k "resnet or skinny or fc" 2>&1 | tail -1
done
for v in "" "MDHB_SKINNY_NW=64" "MDHB_SKINNY_NW=128" "MDHB_SKINNY_NW=64 MDHB_SKINNY_CS=16" "MDHB_SKINNY_NW=128 MDHB_SKINNY_CS=16" "MDHB_SKINNY_NW=128 MDHB_SKINNY_CS=4" ""; do
  echo "FC $v"; env $v timeout 120 python tools/graph_time.py matmul_resnet_fc 400 2>&1 | tail -1 | cut -c1-120
done
