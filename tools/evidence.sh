#!/bin/bash
# Round evidence on one GPU (run under gpurun): GPU tests, the bench line, the
# ncu launch list of the bench command, one ncu --set full summary per routine.
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
bash tools/launch_list.sh
bash tools/profile_all.sh jacobi3d_fp32 matvec_fp32 matmul_fp32 matmul_fp32:tf32 matmul_resnet_fc mcc_nhwc mcc_nhwc:tf32 \
     ccsdt_abcdef_gdab_efgc ccsdt_abcdef_gdab_efgc:tf32 prl_max scan_i32 mcc_nhwc:bf16 matmul_fp32:bf16 ccsdt_abcdef_gdab_efgc:bf16
cat gpurun_out/gpu_tests.log
