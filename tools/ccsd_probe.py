"""Is CCSD(T)'s FFMA time a small-K effect or a layout effect? (dev aid)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh  # noqa: E402

for name, sizes in [("ccsdt_abcdef_gdab_efgc", None), ("matmul_fp32", [13824, 13824, 72]),
                    ("matmul_fp32", [13824, 13824, 80]), ("matmul_fp32", [13824, 13824, 96]),
                    ("matmul_fp32", [13824, 13824, 128]), ("matmul_fp32", [13824, 13824, 256])]:
    j = json.load(open(f"specs/{name}.json"))
    if sizes:
        j["sizes"] = sizes
    p = mdh.Plan(j)
    ins = p.empty(0)
    for t in ins:
        t.uniform_(-1, 1)
    outs = p.empty(1)
    med, _ = p.time(ins, outs, warmup=1, reps=5)
    d = p.describe()
    print(f"{name:24s} {str(j['sizes']):28s} {med * 1e3:8.3f} ms {d['flops'] / med / 1e12:6.2f} TF  {d['template']['kernel']}", flush=True)
