MDHB_STENCIL_S32=53 timeout 300 python -m pytest tests/test_gpu_stencil.py -m gpu -q -x 2>&1 | grep -E "^E|Error|def test" | head -12
