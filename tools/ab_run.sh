for v in "" "MDHB_TC_MC=1"; do
  echo "M $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 10 2>&1 | tail -1 | cut -c1-700
  echo "Mb $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:bf16 10 2>&1 | tail -1 | cut -c1-100
done
