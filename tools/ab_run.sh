timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_tuner_space.py tests/test_gpu_dev_layer.py -m gpu -q 2>&1 | tail -3
for v in "" "MDHB_STENCIL_TI=64" "MDHB_STENCIL_TI=16" "MDHB_STENCIL_TI=128"; do
  echo "J $v"; env $v timeout 120 python tools/graph_time.py jacobi3d_fp32 200 2>&1 | tail -1 | cut -c1-100
done
timeout 600 python bench.py --no-routines > gpurun_out/bench_ab.log 2>&1; tail -c 1500 gpurun_out/bench_ab.log
