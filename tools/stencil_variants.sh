#!/bin/bash
# A/B of stencil kernel variants (development aid)
for rep in 1 2; do
for v in "MDHB_STENCIL_LEAN=54" "MDHB_STENCIL_TS=1" "MDHB_STENCIL_LEAN=44" "MDHB_STENCIL_LEAN=0"; do
  echo -n "$v : "; env $v timeout 60 python bench.py --no-cpu --no-routines --steps 200 | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(d['value'], d['config']['kernel'])"
done
done
