import json, sys, torch
sys.path.insert(0, '.')
from paper_2405_05118_b200 import mdh
for name in ["jacobi3d_fp32", "matvec_fp32"]:
    spec = json.load(open(f"specs/{name}.json"))
    p = mdh.Plan(spec)
    d_in = p.empty(0); [t.uniform_(-1, 1) for t in d_in]
    d_out = p.empty(1)
    med, ker = p.time(d_in, d_out, warmup=3, reps=10, flush_l2=True)
    d = p.describe()
    print(name, d["family"], d["template"], "ms", med * 1e3, "GB/s", d["bytes"] / med / 1e9)
