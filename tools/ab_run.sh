set -x
timeout 600 python -m pytest tests/test_gpu_tuner_space.py tests/test_gpu_contraction.py -m gpu -q -x 2>&1 | tail -3
for v in "" "MDHB_SKINNY_LAST=1" "MDHB_SKINNY_LAST=1 MDHB_SKINNY_CS=16" "MDHB_SKINNY_LAST=1 MDHB_SKINNY_CS=4" "MDHB_SKINNY_CS=16"; do
  echo "FC $v"; env $v timeout 120 python tools/graph_time.py matmul_resnet_fc 400 2>&1 | tail -1
done
for v in "" "MDHB_TC_NO_TRANSPOSE=1"; do
  echo "TF32 $v"; env $v timeout 120 python tools/graph_time.py matmul_fp32:tf32 20 2>&1 | tail -1
done
timeout 300 python -m pytest tests/test_gpu_tc.py -m gpu -q -x -k "matmul" 2>&1 | tail -2
MDHB_TC_NO_TRANSPOSE=1 timeout 300 python -m pytest tests/test_gpu_tc.py -m gpu -q -x -k "matmul" 2>&1 | tail -2
timeout 500 python bench.py --no-routines > gpurun_out/bench_ab.log 2>&1; tail -c 600 gpurun_out/bench_ab.log
