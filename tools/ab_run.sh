# scratch A/B (development aid): K tail (32/64-byte last k-step) on CCSD(T) TF32 / BF16
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_tuner_space.py -m gpu -q -x 2>&1 | tail -2
python - <<'PY'
import json, sys
sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh
j = json.load(open("specs/ccsdt_abcdef_gdab_efgc.json"))
for m in (1, 2):
    print(mdh.Plan(j, math=m).describe()["template"])
PY
for i in 1 2; do
for v in "" "MDHB_TC_NO_KTAIL=1"; do
  echo "C tf32 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:tf32 50 2>&1 | tail -1 | cut -c1-90
  echo "C bf16 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:bf16 50 2>&1 | tail -1 | cut -c1-90
done
done
