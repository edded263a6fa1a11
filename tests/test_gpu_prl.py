"""PRL (max_PRL as a packed key, pw:max) on the prl family: bit-exact vs the
oracle and vs a brute-force argmax with lowest-id tie-break."""
import json

import numpy as np
import pytest

from helpers import run_device, spec
from oracle import mdh_oracle as mo


def brute(Q, D, W, S=1 << 20, C=(1 << 20) - 1):
    wt = ((Q[:, None, :] == D[None, :, :]) * W).sum(-1)
    r = np.arange(D.shape[0])
    return (wt * S + (C - r)[None, :]).max(axis=1)


@pytest.mark.gpu
@pytest.mark.parametrize("nq,nr,vals,istore", [(64, 4096, 3, "i32"), (300, 5000, 3, "i64"), (1024, 2048, 100, "i32"),
                                               (256, 1 << 14, 3, "i64")])
def test_prl_fast_path_bit_exact(nq, nr, vals, istore):
    from paper_2405_05118_b200 import mdh
    j = spec("prl_max", [nq, nr])
    comp = mo.Computation.from_json(j)
    rng = np.random.default_rng(nq + nr)
    Q = rng.integers(0, vals, (nq, 4))
    D = rng.integers(0, vals, (nr, 4))
    W = np.array([3, 5, 7, 9])
    plan = mdh.Plan(j, int_storage=mdh.I32 if istore == "i32" else mdh.I64)
    assert plan.describe()["family"] == "prl"
    (got,) = run_device(plan, [Q, D, W])
    ((want, _),) = mo.execute(comp, [Q, D, W])
    assert np.array_equal(got.astype(np.int64), want)
    assert np.array_equal(want, brute(Q, D, W))


@pytest.mark.gpu
def test_prl_slow_path_wide_values_and_negative_weights():
    """Values outside a 128-wide window / weights beyond a byte: exact 64-bit path."""
    from paper_2405_05118_b200 import mdh
    j = spec("prl_max", [128, 3000])
    comp = mo.Computation.from_json(j)
    rng = np.random.default_rng(5)
    Q = rng.integers(-1000, 1000, (128, 4))
    D = Q[rng.integers(0, 128, 3000)] * (rng.random((3000, 1)) < 0.5) + rng.integers(-1000, 1000, (3000, 4)) * 0
    D[::7] = rng.integers(-1000, 1000, (len(D[::7]), 4))
    W = np.array([300, -2, 7, 1000])
    plan = mdh.Plan(j)
    (got,) = run_device(plan, [Q, D, W])
    ((want, _),) = mo.execute(comp, [Q, D, W])
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_prl_full_size_sampled_queries():
    """2^15 x 2^20 on the device; 48 queries re-checked by the oracle."""
    import torch
    from paper_2405_05118_b200 import mdh
    j = spec("prl_max")
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j, int_storage=mdh.I32)
    g = torch.Generator(device="cuda").manual_seed(3)
    Qd, Dd, Wd = plan.empty(0)
    Qd.random_(0, 3, generator=g)
    Dd.random_(0, 3, generator=g)
    Wd.copy_(torch.tensor([3, 5, 7, 9], dtype=Wd.dtype))
    (out,) = plan.empty(1)
    plan.run([Qd, Dd, Wd], [out])
    torch.cuda.synchronize()
    Q, D, W = (t.cpu().numpy().astype(np.int64) for t in (Qd, Dd, Wd))
    got = out.cpu().numpy()
    for lo in (0, 16384, 32760):
        ((part, _),), sh = mo.execute_box(comp, [Q, D, W], {0: (lo, lo + 8)})
        assert np.array_equal(got[lo:lo + 8], part)
    idx = np.random.default_rng(1).integers(0, 32768, 24)
    assert np.array_equal(got[idx], brute(Q[idx], D, W))


@pytest.mark.gpu
@pytest.mark.parametrize("five", [False, True])
@pytest.mark.parametrize("W", [[3, 20, 7, 9], [3, -2, 7, 9], [0, 15, 1, 15]])
def test_prl_weight_encodings_bit_exact(W, five, monkeypatch):
    """Weights in [0, 15] take the five-instruction path (DP4A yields
    2^11 * wsum + reversed tile index); byte-range weights outside it take the
    six-instruction path; both are bit-exact.  Record counts straddle the
    2048-record tiles and the record splits."""
    from paper_2405_05118_b200 import mdh
    j = spec("prl_max", [300, 2048 * 3 + 77])
    comp = mo.Computation.from_json(j)
    rng = np.random.default_rng(11)
    Q = rng.integers(0, 3, (300, 4))
    D = rng.integers(0, 3, (2048 * 3 + 77, 4))
    W = np.array(W)
    if five:
        monkeypatch.setenv("MDHB_PRL_5", "1")
    plan = mdh.Plan(j, int_storage=mdh.I32)
    (got,) = run_device(plan, [Q, D, W])
    ((want, _),) = mo.execute(comp, [Q, D, W])
    assert np.array_equal(got.astype(np.int64), want)
    assert np.array_equal(want, brute(Q, D, W))
