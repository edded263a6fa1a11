"""Small invocations of the newest kernels for compute-sanitizer runs
(development aid): FFMA conv (TMA ring), tcgen05 conv (pair, single, bf16),
SimCost-free plan paths."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from helpers import run_device, spec  # noqa: E402
from oracle import mdh_oracle as mo  # noqa: E402
from paper_2405_05118_b200 import mdh  # noqa: E402

j = spec("mcc_nhwc", [2, 20, 16, 64, 3, 3, 32])
comp = mo.Computation.from_json(j)
ins = mo.make_inputs(comp, 3)
for math in (mdh.MATH_FFMA, mdh.MATH_TF32, mdh.MATH_BF16):
    p = mdh.Plan(j, math=math)
    (out,) = run_device(p, ins)
    print(p.describe()["template"]["kernel"], float(np.abs(out).sum()))
