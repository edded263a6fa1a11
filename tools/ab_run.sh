for v in "" "MDHB_STENCIL_PF=2" "MDHB_STENCIL_PF=4" "MDHB_STENCIL_PF=8" "" "MDHB_STENCIL_PF=4 MDHB_STENCIL_S32=63"; do
  echo "J $v"; env $v timeout 120 python tools/graph_time.py jacobi3d_fp32 200 2>&1 | tail -1 | cut -c1-60
done
MDHB_STENCIL_PF=4 timeout 300 python -m pytest tests/test_gpu_stencil.py -m gpu -q 2>&1 | tail -1
