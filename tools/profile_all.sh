#!/bin/bash
# One ncu --set full capture per routine (development aid; run under gpurun on
# ONE GPU).  Writes gpurun_out/prof_<routine>.ncu-rep; summarise here with
#   python tools/ncu_summary.py --by-routine gpurun_out <tag>
KRE='regex:star7|gemv|sgemm|skinny|tc_gemm|prl_main|vm_|scan_|layout'
for r in "$@"; do
  f=${r/:/__}
  timeout 600 ncu --set full --clock-control none --import-source on -k "$KRE" -c 6 \
      -o gpurun_out/prof_$f -f python tools/profile_routines.py $r > gpurun_out/prof_$f.log 2>&1
  echo "$r rc=$?"
done
