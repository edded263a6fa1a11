"""Device time of the NVRTC-emitted kernel vs the bytecode VM on md_homs no
specialised family claims (development aid)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh  # noqa: E402

REF = "tests/golden/reference_data/computations"
cases = [("bmatmul", [64, 256, 256, 256]), ("conv2d", [1024, 1024, 5, 5]), ("double_reduce", [1 << 24]),
         ("histo", [1 << 20, 64])]
for name, sizes in cases:
    j = json.load(open(os.path.join(REF, name + ".json")))
    j["sizes"] = sizes
    for generic in (False, True):
        p = mdh.Plan(j, generic=generic)
        ins = p.empty(0)
        for t in ins:
            if t.is_floating_point():
                t.uniform_(-1, 1)
            else:
                t.random_(0, 7)
        outs = p.empty(1)
        med, _ = p.time(ins, outs, warmup=1, reps=3)
        d = p.describe()
        print(f"{name:14s} {str(sizes):24s} {d['family']:8s} {med * 1e3:10.3f} ms  {d['bytes'] / med / 1e9:8.1f} GB/s", flush=True)
