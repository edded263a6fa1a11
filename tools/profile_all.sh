#!/bin/bash
# One ncu --set full capture per routine (development aid; run under gpurun on
# ONE GPU).  On the box each report is reduced to gpurun_out/prof_<routine>.json
# (tools/ncu_summary.py) + .hot.txt (tools/sass_hot.py) and deleted unless
# KEEP_REP=1, so the results fit gpurun's 64 MiB return limit.  Here:
#   python tools/ncu_summary.py --by-routine gpurun_out <tag>
KRE='regex:star7|gemv|sgemm|skinny|tc_gemm|tc_conv|ffma_conv|prl_main|vm_|scan_|layout|pack_|mdh_emitted'
for r in "$@"; do
  f=${r/:/__}
  timeout 600 ncu --set full --clock-control none --import-source on -k "$KRE" -c 8 \
      -o gpurun_out/prof_$f -f python tools/profile_routines.py $r > gpurun_out/prof_$f.log 2>&1
  echo "$r rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_$f.ncu-rep > gpurun_out/prof_$f.json
  python tools/sass_hot.py gpurun_out/prof_$f.ncu-rep 30 > gpurun_out/prof_$f.hot.txt
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_$f.ncu-rep
done
