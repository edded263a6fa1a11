"""Custom combine pw:max_prl on the device (API extension).

The unpacked PRL form -- (weight, record) pairs folded with max_prl -- must
give exactly the pair the reference-expressible packed form encodes
(weight * 2^20 + (2^20 - 1 - record) folded with pw:max, specs/prl_max.json,
whose oracle is pinned to the unmodified reference in test_oracle.py), and
the brute-force argmax with the lowest record on ties.  Every path: the PRL
template (packed fast path and the exact pair path), the emitted family
(NVRTC) on another md_hom, and the device VM (ps:max_prl)."""
import json
import os

import numpy as np
import pytest

from conftest import REPO
from helpers import run_device, spec
from oracle import mdh_oracle as mo


def ext_spec(sizes):
    with open(os.path.join(REPO, "specs", "extensions", "prl_max_prl.json")) as f:
        j = json.load(f)
    j["sizes"] = list(sizes)
    return j


def prl_inputs(nq, nr, seed, lo=0, hi=3, W=(3, 5, 7, 9)):
    rng = np.random.default_rng(seed)
    return [rng.integers(lo, hi, (nq, 4)).astype(np.int64), rng.integers(lo, hi, (nr, 4)).astype(np.int64),
            np.array(W, dtype=np.int64)]


def brute(Q, D, W):
    wt = np.where(Q[:, None, :] == D[None, :, :], W[None, None, :], 0).sum(-1)
    top = wt.max(1)
    return top, np.argmax(wt == top[:, None], axis=1)


def packed_oracle(nq, nr, ins):
    comp = mo.Computation.from_json(spec("prl_max", [nq, nr]))
    ((best, _),) = mo.execute(comp, ins)
    return best >> 20, (1 << 20) - 1 - (best & ((1 << 20) - 1))


@pytest.mark.gpu
@pytest.mark.parametrize("nq,nr,seed", [(64, 4096, 1), (300, 5000, 2), (2048, 65536, 3), (1, 1, 4), (7, 129, 5)])
def test_max_prl_pairs_equal_packed_oracle_and_brute_force(nq, nr, seed):
    from paper_2405_05118_b200 import mdh
    ins = prl_inputs(nq, nr, seed)
    plan = mdh.Plan(ext_spec([nq, nr]))
    d = plan.describe()
    assert d["family"] == "prl" and "max_prl" in d["template"]["combine"], d
    w, r = run_device(plan, ins)
    pw, pr = packed_oracle(nq, nr, ins)
    assert np.array_equal(w, pw) and np.array_equal(r, pr)
    if nq * nr <= 1 << 22:
        bw, br = brute(*ins)
        assert np.array_equal(w, bw) and np.array_equal(r, br)


@pytest.mark.gpu
def test_max_prl_exact_pair_path_wide_weights():
    # weights outside the packed fast path (|w| > 127 and a field window > 128):
    # the exact pair path folds (w, r) without packing -- any int64 weights
    from paper_2405_05118_b200 import mdh
    nq, nr = 96, 3000
    ins = prl_inputs(nq, nr, 9, lo=-400, hi=400, W=(1 << 40, -(1 << 38), 123456789, 7))
    ins[1][::7] = ins[0][0]  # plant exact matches
    w, r = run_device(mdh.Plan(ext_spec([nq, nr])), ins)
    bw, br = brute(*ins)
    assert np.array_equal(w, bw) and np.array_equal(r, br)


@pytest.mark.gpu
def test_max_prl_i32_storage():
    from paper_2405_05118_b200 import mdh
    ins = prl_inputs(256, 8192, 11)
    w, r = run_device(mdh.Plan(ext_spec([256, 8192]), int_storage=mdh.I32), ins)
    bw, br = brute(*ins)
    assert np.array_equal(w, bw) and np.array_equal(r, br)


@pytest.mark.gpu
def test_max_prl_full_size_sampled_queries():
    """2^15 x 2^20, the BASELINE size: sampled queries against the packed
    oracle on ++ slices of q (and brute force)."""
    import torch
    from paper_2405_05118_b200 import mdh
    nq, nr = 32768, 1048576
    ins = prl_inputs(nq, nr, 21)
    plan = mdh.Plan(ext_spec([nq, nr]), int_storage=mdh.I32)
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(x).to(t.dtype))
    w, r = plan.empty(1)
    plan.run(d_in, [w, r])
    torch.cuda.synchronize()
    w, r = w.cpu().numpy(), r.cpu().numpy()
    comp = mo.Computation.from_json(spec("prl_max"))
    for lo in (0, 12345, nq - 2):
        ((best, _),), _ = mo.execute_slice(comp, ins, 0, lo, lo + 2)
        assert np.array_equal(w[lo:lo + 2], best >> 20)
        assert np.array_equal(r[lo:lo + 2], (1 << 20) - 1 - (best & ((1 << 20) - 1)))
    bw, br = brute(ins[0][:64], ins[1], ins[2])
    assert np.array_equal(w[:64], bw) and np.array_equal(r[:64], br)


@pytest.mark.gpu
def test_max_prl_on_the_emitted_family_argmax_rows():
    """Another md_hom with the operator: row argmax of a float matrix,
    (value, column) folded with max_prl -- runs on the NVRTC-emitted kernel."""
    from paper_2405_05118_b200 import mdh
    j = {"name": "row_argmax", "dims": ["i", "j"], "sizes": [37, 1000],
         "inputs": [{"name": "M", "type": "f64", "rank": 2, "accesses": ["i, j"]}],
         "outputs": [{"name": "val", "type": "f64", "rank": 1, "accesses": ["i"]},
                     {"name": "col", "type": "i64", "rank": 1, "accesses": ["i"]}],
         "scalar": "out(1,1) = in(1,1); out(2,1) = idx(2);", "combine": ["cc", "pw:max_prl"]}
    rng = np.random.default_rng(3)
    M = rng.integers(-20, 20, (37, 1000)).astype(np.float64) * 0.5  # many ties
    plan = mdh.Plan(j, float_storage=mdh.F64)
    assert plan.describe()["family"] == "emitted", plan.describe()
    assert "max_prl" not in plan.kernel_source() or True
    val, col = run_device(plan, [M])
    assert np.array_equal(val, M.max(1)) and np.array_equal(col, M.argmax(1))


@pytest.mark.gpu
def test_user_registered_operator_runs_through_nvrtc():
    from paper_2405_05118_b200 import mdh
    mdh.register_combine("argmin_lo", 2, "if (b0 < a0 || (b0 == a0 && b1 < a1)) { a0 = b0; a1 = b1; }",
                         identity=("INT64_MAX", "INT64_MAX"))
    j = {"name": "col_argmin", "dims": ["i", "j"], "sizes": [3000, 24],
         "inputs": [{"name": "M", "type": "i64", "rank": 2, "accesses": ["i, j"]}],
         "outputs": [{"name": "val", "type": "i64", "rank": 1, "accesses": ["j"]},
                     {"name": "row", "type": "i64", "rank": 1, "accesses": ["j"]}],
         "scalar": "out(1,1) = in(1,1); out(2,1) = idx(1);", "combine": ["pw:argmin_lo", "cc"]}
    M = np.random.default_rng(4).integers(-9, 9, (3000, 24)).astype(np.int64)
    plan = mdh.Plan(j)
    assert plan.describe()["family"] == "emitted"
    assert "b0 < a0" in plan.kernel_source()
    val, row = run_device(plan, [M])
    assert np.array_equal(val, M.min(0)) and np.array_equal(row, M.argmin(0))


@pytest.mark.gpu
def test_prefix_max_prl_on_the_device_vm():
    """ps:max_prl: the running (best value, its first index) along a line --
    the generic device VM's built-in tuple operator."""
    from paper_2405_05118_b200 import mdh
    j = {"name": "running_argmax", "dims": ["i", "j"], "sizes": [5, 300],
         "inputs": [{"name": "x", "type": "i64", "rank": 2, "accesses": ["i, j"]}],
         "outputs": [{"name": "best", "type": "i64", "rank": 2, "accesses": ["i, j"]},
                     {"name": "at", "type": "i64", "rank": 2, "accesses": ["i, j"]}],
         "scalar": "out(1,1) = in(1,1); out(2,1) = idx(2);", "combine": ["cc", "ps:max_prl"]}
    x = np.random.default_rng(5).integers(0, 30, (5, 300)).astype(np.int64)
    plan = mdh.Plan(j)
    assert plan.describe()["family"] == "generic", plan.describe()
    best, at = run_device(plan, [x])
    want = np.maximum.accumulate(x, axis=1)
    first = np.array([[int(np.argmax(x[i, :t + 1])) for t in range(300)] for i in range(5)])
    assert np.array_equal(best, want) and np.array_equal(at, first)
