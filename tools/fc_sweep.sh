# FC cluster-size sweep (development aid)
for i in 1 2; do
for v in "X=1" "MDHB_SKINNY_CS=4" "MDHB_SKINNY_CS=16"; do
  echo "$v $(env $v python tools/graph_time.py matmul_resnet_fc 200 2>&1 | tail -1 | cut -c1-70)"
done; done
