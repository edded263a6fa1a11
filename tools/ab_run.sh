MDHB_STENCIL_T1D=44 timeout 300 python -m pytest tests/test_gpu_stencil.py -m gpu -q -x 2>&1 | grep -E "Error|error|assert|^E" | head -20
MDHB_STENCIL_T1D=44 timeout 120 python tools/graph_time.py jacobi3d_fp32 20 2>&1 | tail -5
