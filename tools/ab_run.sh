# scratch A/B (development aid): FFMA defaults vs alternatives on this box
for i in 1 2; do
for v in "" "MDHB_PIPE_128x128=1"; do
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-80
done
for v in "" "MDHB_FFMA_CONV=1"; do
  echo "F $v"; env $v timeout 120 python tools/graph_time.py mcc_nhwc 10 2>&1 | tail -1 | cut -c1-80
done
done
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm,pci.bus_id --format=csv
