"""Jacobi3D (BASELINE config 2) on the stencil family vs the oracle."""
import numpy as np
import pytest

from helpers import assert_close, run_device, spec, uniform_inputs
from oracle import mdh_oracle as mo


@pytest.mark.gpu
@pytest.mark.parametrize("sizes", [[8, 8, 16], [3, 16, 128], [5, 32, 256], [7, 20, 130], [40, 48, 384], [6, 8, 256],
                                   [5, 4, 512], [9, 12, 512], [4, 20, 256]])
def test_jacobi3d_small_vs_oracle(sizes):
    from paper_2405_05118_b200 import mdh
    j = spec("jacobi3d_fp32", sizes)
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j)
    d = plan.describe()
    assert d["family"] == "stencil", d
    ins = uniform_inputs(comp, 1)
    got = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert_close(got[0], want, dfd, 7, f"jacobi3d {sizes}")


@pytest.mark.gpu
def test_jacobi3d_full_size_slices_vs_oracle():
    """512^3 output: first, middle and last i-planes checked against the oracle
    run on ++-slices (the homomorphic property), the rest via linearity."""
    import torch
    from paper_2405_05118_b200 import mdh
    j = spec("jacobi3d_fp32")
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j)
    assert plan.describe()["family"] == "stencil"
    g = torch.Generator(device="cuda").manual_seed(7)
    (v,) = plan.empty(0)
    v.uniform_(-1, 1, generator=g)
    (w,) = plan.empty(1)
    plan.run([v], [w])
    # linearity: f(2v) == 2 f(v) exactly in fp32 (scaling by 2 is exact)
    (w2,) = plan.empty(1)
    plan.run([v * 2], [w2])
    torch.cuda.synchronize()
    assert torch.equal(w2, 2 * w)
    vh = v.cpu().numpy().astype(np.float64)
    for lo in (0, 255, 510):
        ((part, dfd),), shifts = mo.execute_slice(comp, [vh], 0, lo, lo + 2)
        got = w[lo:lo + 2].cpu().numpy()
        assert_close(got, part, dfd, 7, f"planes {lo}..{lo + 2}")


@pytest.mark.gpu
@pytest.mark.parametrize("sizes", [[40, 48, 384], [512, 512, 512]])
def test_jacobi3d_host_pipeline_equals_device_run(sizes):
    """mdh_b200_run_host (chunked H2D / compute / D2H overlap along i) gives
    exactly the device-resident result."""
    import torch
    from paper_2405_05118_b200 import mdh
    j = spec("jacobi3d_fp32", sizes)
    plan = mdh.Plan(j)
    (v,) = plan.empty(0)
    v.uniform_(-1, 1)
    (w,) = plan.empty(1)
    plan.run([v], [w])
    torch.cuda.synchronize()
    vh = v.cpu().pin_memory()
    wh = torch.empty(w.shape, dtype=w.dtype).pin_memory()
    plan.run_host([vh.numpy()], [wh.numpy()])
    assert torch.equal(wh, w.cpu())


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["0", "63", "44", "54", "ts"])
def test_jacobi3d_variants_bit_identical(env, monkeypatch):
    """Every stencil kernel variant (star7_ws, the packed-lane lean rings, the
    TMA-store epilogue) computes the default's (star7_s32) bits: same FMA
    order per output cell."""
    from paper_2405_05118_b200 import mdh
    j = spec("jacobi3d_fp32", [40, 48, 384])
    comp = mo.Computation.from_json(j)
    ins = uniform_inputs(comp, 5)
    p0 = mdh.Plan(j)
    assert p0.describe()["template"]["kernel"] == "star7_s32<5,3>", p0.describe()
    (base,) = run_device(p0, ins)
    if env == "ts":
        monkeypatch.setenv("MDHB_STENCIL_TS", "1")  # TMA bulk stores (full tiles: 48 x 384 qualify)
    else:
        monkeypatch.setenv("MDHB_STENCIL_LEAN", env)
    plan = mdh.Plan(j)
    assert plan.describe()["template"]["kernel"].startswith("star7_ws" if env == "0" else "star7_lean"), plan.describe()
    (var,) = run_device(plan, ins)
    assert np.array_equal(base, var)
