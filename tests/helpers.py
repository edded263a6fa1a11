"""Shared helpers for the parity tests: run an md_hom through the B200 C ABI
and the oracle on identical inputs."""
import json
import os

import numpy as np

from conftest import GOLDEN, REPO

SPECS = os.path.join(REPO, "specs")
REFDATA = os.path.join(GOLDEN, "reference_data")


def spec(name, sizes=None):
    with open(os.path.join(SPECS, name + ".json")) as f:
        j = json.load(f)
    if sizes is not None:
        j["sizes"] = list(sizes)
    return j


def bundled(name, sizes=None):
    with open(os.path.join(REFDATA, "computations", name + ".json")) as f:
        j = json.load(f)
    if sizes is not None:
        j["sizes"] = list(sizes)
    return j


def run_device(plan, inputs):
    """Copies numpy inputs into device tensors of the plan's storage types,
    runs mdh_b200_run on the current stream, returns numpy outputs."""
    import torch
    d_in = plan.empty(0)
    for t, x in zip(d_in, inputs):
        t.copy_(torch.from_numpy(np.ascontiguousarray(x)).to(t.dtype))
    d_out = plan.empty(1)
    for t in d_out:
        t.zero_()
    plan.run(d_in, d_out)
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in d_out]


def exact_inputs(comp, seed):
    """The reference's own generator (support.hpp:32-51): k/4 floats, |k|<=5."""
    from oracle import mdh_oracle as mo
    return mo.make_inputs(comp, seed)


def uniform_inputs(comp, seed):
    from oracle import mdh_oracle as mo
    rng = np.random.default_rng(seed)
    out = []
    for vb, shp in zip(comp.inputs, mo.input_shapes(comp)):
        if vb.type == "f64":
            out.append(rng.uniform(-1, 1, shp).astype(np.float32).astype(np.float64))
        else:
            out.append(rng.integers(-5, 6, shp).astype(np.int64))
    return out


def assert_close(got, want, defined, K, what=""):
    """FP32 parity bound of north_star: |d| <= 1e-5 * sqrt(K) * max(|ref|, 1)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    m = np.asarray(defined, dtype=bool)
    tol = 1e-5 * np.sqrt(max(K, 1)) * np.maximum(np.abs(want), 1.0)
    bad = (np.abs(got - want) > tol) & m
    assert not bad.any(), f"{what}: {bad.sum()} cells out of tolerance, e.g. got {got[bad][:4]} want {want[bad][:4]}"
