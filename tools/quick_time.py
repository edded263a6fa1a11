"""Quick per-routine timing through the C ABI (development aid, not the bench)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh  # noqa: E402

names = sys.argv[1:] or ["jacobi3d_fp32", "matvec_fp32", "matmul_fp32", "matmul_resnet_fc", "mcc_nhwc",
                         "ccsdt_abcdef_gdab_efgc", "prl_max"]
for name in names:
    math = mdh.MATH_FFMA
    if ":" in name:
        name, m = name.split(":")
        math = {"tf32": mdh.MATH_TF32, "bf16": mdh.MATH_BF16}[m]
    spec = json.load(open(f"specs/{name}.json"))
    try:
        p = mdh.Plan(spec, math=math, int_storage=mdh.I32)
    except mdh.MdhError as e:
        print(name, "ERROR", e)
        continue
    d_in = p.empty(0)
    for t in d_in:
        if t.is_floating_point():
            t.uniform_(-1, 1)
        else:
            t.random_(0, 3)
    d_out = p.empty(1)
    reps = 3 if name in ("matmul_fp32", "prl_max") else 10
    med, ker = p.time(d_in, d_out, warmup=2, reps=reps, flush_l2=True)
    d = p.describe()
    print(f"{name:26s} {d['family']:12s} {med*1e3:9.4f} ms  {d['bytes']/med/1e9:8.1f} GB/s  "
          f"{d['flops']/med/1e12:7.2f} TFLOP/s  {json.dumps(d['template'])}", flush=True)
