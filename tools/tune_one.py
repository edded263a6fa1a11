"""Run the on-device tuner on one BASELINE spec and print the history."""
import json
import sys

sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh  # noqa: E402

name = sys.argv[1]
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = json.load(open(f"specs/{name}.json"))
best, hist, secs = mdh.tune(json.dumps(spec), "B200", budget=budget, seed=0, int_storage=mdh.I32)
print(hist)
print("best seconds", secs)
p = mdh.Plan(spec, "B200", best, int_storage=mdh.I32)
print(json.dumps(p.describe()["template"]))
