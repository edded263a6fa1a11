timeout 600 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_tuner_space.py -m gpu -q -x -k "stencil or jacobi" 2>&1 | tail -2
for v in "" "MDHB_STENCIL_S32=63" "MDHB_STENCIL_S32=73" "MDHB_STENCIL_LEAN=54" "" "MDHB_STENCIL_S32=63"; do
  echo "J $v"; env $v timeout 120 python tools/graph_time.py jacobi3d_fp32 200 2>&1 | tail -1 | cut -c1-60
done
