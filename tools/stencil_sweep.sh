#!/bin/bash
# stencil variants (development aid)
for v in "X=1" "MDHB_STENCIL_TI=16" "MDHB_STENCIL_TI=64" "MDHB_STENCIL_TI=128" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=2" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3" \
         "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3 MDHB_STENCIL_TI=16" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3 MDHB_STENCIL_TI=64" \
         "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=3 MDHB_STENCIL_RANGES=1" "MDHB_STENCIL_PERS=1 MDHB_STENCIL_MINB=2 MDHB_STENCIL_RANGES=1"; do
  echo -n "$v : "; env $v timeout 60 python bench.py --no-cpu --no-routines --steps 100 | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(d['value'], d['config']['kernel'])"
done
