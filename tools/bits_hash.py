"""Hash of one routine's output on seeded U(-1,1) inputs (development aid:
compare env-selected variants bit for bit).  Usage: python tools/bits_hash.py name[:tf32|:bf16] [sizes...]"""
import hashlib
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh  # noqa: E402

name = sys.argv[1]
math = mdh.MATH_FFMA
if ":" in name:
    name, m = name.split(":")
    math = {"tf32": mdh.MATH_TF32, "bf16": mdh.MATH_BF16}[m]
spec = json.load(open(f"specs/{name}.json"))
if len(sys.argv) > 2:
    spec["sizes"] = [int(x) for x in sys.argv[2:]]
p = mdh.Plan(spec, math=math, int_storage=mdh.I32)
torch.manual_seed(7)
d_in = p.empty(0)
for t in d_in:
    t.copy_(torch.rand(t.shape, dtype=torch.float32).mul_(2).sub_(1).to(t.dtype))
d_out = p.empty(1)
for t in d_out:
    t.fill_(float("nan"))
p.run(d_in, d_out)
torch.cuda.synchronize()
h = hashlib.sha256()
for t in d_out:
    h.update(t.cpu().numpy().tobytes())
print(name, spec["sizes"], p.describe()["template"]["kernel"], h.hexdigest()[:16])
