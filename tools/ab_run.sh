MDHB_STENCIL_TKC=512 timeout 300 python -m pytest tests/test_gpu_stencil.py -m gpu -q 2>&1 | grep -E "^E|^FAILED" | head -30
