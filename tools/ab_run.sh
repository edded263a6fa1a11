# scratch (development aid): FFMA Table-1 instances, contraction parity, timings
timeout 900 python -m pytest tests/test_gpu_tuner_space.py tests/test_gpu_contraction.py tests/test_gpu_fullsize.py tests/test_gpu_tuner.py -m gpu -q -x 2>&1 | tail -3
python - <<'PY'
import json, sys
sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh
for n in ("matmul_fp32", "ccsdt_abcdef_gdab_efgc"):
    j = json.load(open(f"specs/{n}.json"))
    print(n, len(mdh.tune_space(j, "contraction")), mdh.Plan(j).describe()["template"])
PY
for i in 1 2; do
  echo "C"; timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc 20 2>&1 | tail -1 | cut -c1-80
  echo "M"; timeout 120 python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-80
done
