"""TF32 tensor-core sweep: operand majorness and tile width (development aid)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_05118_b200 import mdh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
base = {"dims": ["i", "j", "k"], "sizes": [n, n, n],
        "outputs": [{"name": "C", "type": "f64", "rank": 2, "accesses": ["i, j"]}],
        "scalar": "out(1,1) = in(1,1) * in(2,1);", "combine": ["cc", "cc", "pw:+"]}
variants = {
    "NN (B[k][n], MN-major)": [{"name": "A", "type": "f64", "rank": 2, "accesses": ["i, k"]},
                               {"name": "B", "type": "f64", "rank": 2, "accesses": ["k, j"]}],
    "NT (B[n][k], K-major)": [{"name": "A", "type": "f64", "rank": 2, "accesses": ["i, k"]},
                              {"name": "B", "type": "f64", "rank": 2, "accesses": ["j, k"]}],
}
for label, ins in variants.items():
    for bn in ("256", "128"):
        os.environ["MDHB_TC_BN"] = bn
        spec = dict(base, name="mm", inputs=ins)
        p = mdh.Plan(spec, math=mdh.MATH_TF32)
        d_in = p.empty(0)
        for t in d_in:
            t.uniform_(-1, 1)
        d_out = p.empty(1)
        med, _ = p.time(d_in, d_out, warmup=2, reps=5)
        d = p.describe()
        print(f"{label:28s} BN={bn}: {med*1e3:8.3f} ms  {d['flops']/med/1e12:7.1f} TFLOP/s  {d['template']['kernel']}", flush=True)
        del p, d_in, d_out
        torch.cuda.empty_cache()
