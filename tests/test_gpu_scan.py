"""Scan family (ps:op prefix dims) vs the oracle's prefix pass
(engine.cpp:337-353).  Integer outputs bit-exact for every op; float storage
within the FP32 tolerance (a parallel scan re-associates the sum)."""
import numpy as np
import pytest

from helpers import assert_close, bundled, exact_inputs, run_device, spec
from oracle import mdh_oracle as mo


def _plan(j, **kw):
    from paper_2405_05118_b200 import mdh
    return mdh.Plan(j, **kw)


def _check_exact(j, kernel, seed=3, **kw):
    comp = mo.Computation.from_json(j)
    plan = _plan(j, **kw)
    d = plan.describe()
    assert d["family"] == "scan" and d["template"]["kernel"].startswith(kernel), d
    ins = exact_inputs(comp, seed)
    got = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got[0].astype(np.int64)[dfd], want.astype(np.int64)[dfd])


@pytest.mark.gpu
@pytest.mark.parametrize("sizes,kernel", [([16], "scan_lines"), ([3000], "scan_lines"), ([5000], "scan_tiles"), ([100000], "scan_tiles"),
                                          ([4096 * 7 + 3], "scan_tiles")])
def test_scan_1d_exact(sizes, kernel):
    _check_exact(bundled("scan", sizes), kernel)


@pytest.mark.gpu
@pytest.mark.parametrize("sizes", [[8, 8], [300, 1000], [1000, 33]])
def test_mbbs_strided_scan_exact(sizes):
    """mbbs: ps over rows through the reversed view "7-i, j" (negative stride)."""
    j = bundled("mbbs", sizes)
    j["inputs"][0]["accesses"] = [f"{sizes[0] - 1}-i, j"]
    _check_exact(j, "scan_lines")


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["+", "min", "max", "*"])
def test_scan_ops_multiline_tiles_exact(op):
    """Several lines of decoupled look-back tiles (ps on the contiguous dim)."""
    j = bundled("mbbs", [3, 20000])
    j["inputs"][0]["accesses"] = ["i, j"]
    j["combine"] = ["cc", f"ps:{op}"]
    if op == "*":  # keep products bounded: inputs in {-1, 1}
        comp = mo.Computation.from_json(j)
        ins = [np.where(np.random.default_rng(1).integers(0, 2, s) == 0, -1, 1).astype(np.int64)
               for s in mo.input_shapes(comp)]
        plan = _plan(j)
        assert plan.describe()["template"]["kernel"].startswith("scan_tiles")
        got = run_device(plan, ins)
        ((want, dfd),) = mo.execute(comp, ins)
        assert np.array_equal(got[0][dfd], want[dfd])
        return
    _check_exact(j, "scan_tiles")


@pytest.mark.gpu
def test_scan_i32_storage_exact():
    from paper_2405_05118_b200 import mdh
    _check_exact(bundled("scan", [50000]), "scan_tiles", int_storage=mdh.I32)


@pytest.mark.gpu
def test_scan_f32_within_tolerance():
    j = bundled("scan", [100000])
    j["inputs"][0]["type"] = j["outputs"][0]["type"] = "f64"
    comp = mo.Computation.from_json(j)
    plan = _plan(j)
    assert plan.describe()["family"] == "scan"
    ins = [np.random.default_rng(4).uniform(-1, 1, s).astype(np.float32).astype(np.float64) for s in mo.input_shapes(comp)]
    got = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert_close(got[0], want, dfd, 100000, "scan f32")


@pytest.mark.gpu
def test_scan_full_size_differences():
    """2^28 int32 elements: y[0] = x[0] and y[t] - y[t-1] = x[t] (mod 2^32) for
    every t -- the size-independent property of a prefix sum."""
    import torch
    from paper_2405_05118_b200 import mdh
    j = spec("scan_i32")
    plan = mdh.Plan(j, int_storage=mdh.I32)
    assert plan.describe()["template"]["kernel"].startswith("scan_tiles")
    (x,) = plan.empty(0)
    x.random_(-1000, 1000)
    (y,) = plan.empty(1)
    plan.run([x], [y])
    torch.cuda.synchronize()
    assert int(y[0]) == int(x[0])
    d = (y[1:].to(torch.int64) - y[:-1].to(torch.int64)) & 0xffffffff
    assert torch.equal(d, x[1:].to(torch.int64) & 0xffffffff)
