#!/bin/bash
# compute-sanitizer memcheck over the GPU tests at their small shapes (run under gpurun)
K="not full and not 8192 and not images and not slices and not 56"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest \
  tests/test_gpu_contraction.py tests/test_gpu_scan.py tests/test_gpu_prl.py -x -q -k "$K"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest \
  tests/test_gpu_tc.py tests/test_gpu_stencil.py tests/test_gpu_generic.py -x -q -k "$K"
# round-2 paths: DEV layer (shared-device shards, peer combine, halo exchange),
# custom combine (128-bit CAS, NVRTC tuple fold, VM), Table-1 instances
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest \
  tests/test_gpu_dev_layer.py tests/test_gpu_custom_combine.py -x -q -k "not world2 and not full_size"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest \
  tests/test_gpu_tuner_space.py -x -q -k "stencil or resident or ffma"
