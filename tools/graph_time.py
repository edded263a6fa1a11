"""Graph-replayed device time of one routine (bench.py's time_device: K runs
from one CUDA graph, inputs rotated past L2) -- development aid for A/B runs
of env-selected variants.  Usage: python tools/graph_time.py name[:tf32|:bf16] [steps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2405_05118_b200 import mdh  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
math = mdh.MATH_FFMA
if ":" in name:
    name, m = name.split(":")
    math = {"tf32": mdh.MATH_TF32, "bf16": mdh.MATH_BF16}[m]
spec = json.load(open(f"specs/{name}.json"))
p = mdh.Plan(spec, math=math, int_storage=mdh.I32)
d_in = p.empty(0)
for t in d_in:
    if t.is_floating_point():
        t.uniform_(-1, 1)
    else:
        t.random_(0, 3)
d_out = p.empty(1)
in_bytes = sum(t.numel() * t.element_size() for t in d_in)
tot, copies = bench.time_device(p, d_in, d_out, steps, 5, in_bytes < bench.L2_BYTES)
print(f"{name} {tot / steps * 1e6:.2f} us/run  copies={copies}  {json.dumps(p.describe()['template'])[:160]}")
