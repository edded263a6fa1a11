#!/bin/bash
# stencil variants (development aid)
for v in "X=1" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=2" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3" \
         "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=2 MDHB_STENCIL_TI=16" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3 MDHB_STENCIL_TI=16" \
         "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3 MDHB_STENCIL_TI=8" "MDHB_STENCIL_TI=16" "MDHB_STENCIL_TI=64"; do
  echo -n "$v : "; env $v timeout 60 python tools/quick_time.py jacobi3d_fp32 | cut -c1-80
done
