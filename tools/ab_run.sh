# scratch sweep (development aid): raster group of the wide CTA-pair GEMM
for i in 1 2; do
for v in "MDHB_TC_GROUP=2" "MDHB_TC_GROUP=4" "" "MDHB_TC_GROUP=16" "MDHB_TC_GROUP=32"; do
  echo "M tf32 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 10 2>&1 | tail -1 | cut -c1-60
  echo "M bf16 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:bf16 10 2>&1 | tail -1 | cut -c1-60
done
done
