import json, sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2405_05118_b200 import mdh
for g in (72, 144, 288, 576):
    spec = json.load(open("specs/ccsdt_abcdef_gdab_efgc.json"))
    spec["sizes"][-1] = g
    p = mdh.Plan(spec, math=mdh.MATH_FFMA, int_storage=mdh.I32)
    d_in = p.empty(0)
    for t in d_in:
        t.uniform_(-1, 1)
    d_out = p.empty(1)
    tot, copies = bench.time_device(p, d_in, d_out, 10, 3, True)
    flops = 2 * 24**6 * g
    us = tot / 10 * 1e6
    print(g, f"{us:.1f} us", f"{flops / (tot / 10) / 1e12:.2f} TF", f"frac {flops / (tot/10) / (148*128*2*1.965e9):.3f}", p.describe()["template"]["kernel"])
