#!/bin/bash
# compute-sanitizer memcheck over the GPU tests at their small shapes (run under gpurun)
K="not full and not 8192 and not images and not slices and not 56"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest \
  tests/test_gpu_contraction.py tests/test_gpu_scan.py tests/test_gpu_prl.py -x -q -k "$K"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest \
  tests/test_gpu_tc.py tests/test_gpu_stencil.py tests/test_gpu_generic.py -x -q -k "$K"
