"""Full BASELINE sizes through every arithmetic (FFMA / TF32 / BF16), checked
against the oracle on ++ slices (the homomorphic property, test_highlevel.cpp
:203-221; slicing itself is pinned to the unmodified reference in
test_oracle.py).

Two input modes, as SURVEY 8(c) states them:
  exact    the reference's generator (k/4, |k| <= 5): every product and
           partial sum is exact in FP32 / TF32 / BF16 -> bit-identical;
  uniform  U(-1,1) rounded to FP32 (the oracle sees the same values widened):
           FFMA  |d| <= 1e-5 * sqrt(K) * max(|ref|, 1)      (north_star)
           TF32  |d_ij| <= 2^-9 * sum_k |a_ik| |b_kj|
           BF16  |d_ij| <= 2^-8 * sum_k |a_ik| |b_kj|
           (sum|a||b| computed by the oracle on |A|, |B| over the same slice).
"""
import numpy as np
import pytest

from helpers import assert_close, exact_inputs, spec, uniform_inputs
from oracle import mdh_oracle as mo

MATHS = {"ffma": 0, "tf32": 1, "bf16": 2}

# routine -> (boxes of cc dims checked, contraction length K)
BOXES = {
    "matmul_fp32": ([{0: (0, 1)}, {0: (8191, 8192)}], 8192),
    "mcc_nhwc": ([{0: (0, 1)}, {0: (255, 256)}], 576),
    "ccsdt_abcdef_gdab_efgc": ([{0: (0, 1), 1: (0, 2)}, {0: (23, 24), 3: (22, 24)}], 72),
}


def _run_full(name, math, ins):
    import torch
    from paper_2405_05118_b200 import mdh
    j = spec(name)
    plan = mdh.Plan(j, math=MATHS[math])
    d = plan.describe()
    assert d["family"] == "contraction", d
    if math != "ffma":
        assert d["template"].get("math") == math, d
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(np.ascontiguousarray(x)).to(t.dtype))
    del ins
    (out,) = plan.empty(1)
    out.fill_(float("nan"))
    plan.run(d_in, [out])
    torch.cuda.synchronize()
    del d_in
    return out, d


def _slice(out, shifts, part):
    sl = tuple(slice(s, s + n) for s, n in zip(shifts[0], part.shape))
    return out[sl].cpu().numpy().astype(np.float64)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(BOXES))
@pytest.mark.parametrize("math", ["ffma", "tf32", "bf16"])
def test_full_size_exact_mode(name, math):
    comp = mo.Computation.from_json(spec(name))
    ins = exact_inputs(comp, 21)
    out, d = _run_full(name, math, ins)
    for box in BOXES[name][0]:
        ((part, dfd),), shifts = mo.execute_box(comp, ins, box)
        got = _slice(out, shifts, part)
        assert np.array_equal(got[dfd], part[dfd]), (name, math, box, d["template"]["kernel"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(BOXES))
@pytest.mark.parametrize("math", ["ffma", "tf32", "bf16"])
def test_full_size_uniform_mode(name, math):
    comp = mo.Computation.from_json(spec(name))
    ins = uniform_inputs(comp, 22)
    out, d = _run_full(name, math, ins)
    K = BOXES[name][1]
    for box in BOXES[name][0]:
        ((part, dfd),), shifts = mo.execute_box(comp, ins, box)
        got = _slice(out, shifts, part)
        assert np.isfinite(got[dfd]).all()
        if math == "ffma":
            assert_close(got, part, dfd, K, f"{name} ffma {box}")
        else:
            ((absw, _),), _ = mo.execute_box(comp, [np.abs(x) for x in ins], box)
            u = 2.0 ** -9 if math == "tf32" else 2.0 ** -8
            err = np.abs(got - part)
            ok = (err <= u * absw + 1e-30)[dfd]
            assert ok.all(), (name, math, box, float((err / np.maximum(absw, 1e-30)).max()))
