"""The on-device auto-tuner (mdh_b200_tune): budget-exact history in the
reference's CSV format, deterministic per seed, best config re-instantiates
and stays correct."""
import json

import numpy as np
import pytest

from helpers import run_device, spec, uniform_inputs
from oracle import mdh_oracle as mo


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes", [("jacobi3d_fp32", [64, 64, 256]), ("prl_max", [4096, 1 << 16]),
                                        ("matmul_fp32", [256, 256, 128])])
def test_tune_history_and_best(name, sizes):
    from paper_2405_05118_b200 import mdh
    j = json.dumps(spec(name, sizes))
    best, hist, secs = mdh.tune(j, "B200", budget=6, seed=1, int_storage=mdh.I32)
    rows = hist.strip().splitlines()
    assert rows[0] == "eval_index,config_hash,objective,valid"
    assert len(rows) == 1 + 6
    assert secs > 0
    assert mdh.validate_config(j, "B200", best) == ""
    plan = mdh.Plan(j, "B200", best, int_storage=mdh.I32)
    comp = mo.Computation.from_json(j)
    if name == "prl_max":
        rng = np.random.default_rng(0)
        ins = [rng.integers(0, 3, (sizes[0], 4)), rng.integers(0, 3, (sizes[1], 4)), np.array([3, 5, 7, 9])]
        (got,) = run_device(plan, ins)
        idx = np.arange(0, sizes[0], 512)
        ((want, _),), _ = mo.execute_box(comp, ins, {0: (0, 8)})
        assert np.array_equal(got[:8], want)
    else:
        ins = uniform_inputs(comp, 1)
        (got,) = run_device(plan, ins)
        ((want, dfd),) = mo.execute(comp, ins)
        assert np.allclose(got[dfd], want[dfd], rtol=1e-4, atol=1e-4)


@pytest.mark.gpu
def test_tvm_gpu_fixture_runs_through_config():
    """The published TVM CUDA schedule (data/fixtures/tvm_gpu.json) on the
    ResNet-50 FC MatMul: accepted, executed, exact."""
    import os
    from conftest import GOLDEN
    from paper_2405_05118_b200 import mdh
    fx = json.load(open(os.path.join(GOLDEN, "reference_data", "fixtures", "tvm_gpu.json")))
    comp_j = json.load(open(os.path.join(GOLDEN, "reference_data", "computations", "matmul_resnet.json")))
    comp_j["sizes"] = fx["sizes"]
    for b in comp_j["inputs"] + comp_j["outputs"]:
        b["type"] = "f64"
    plan = mdh.Plan(comp_j, fx["model"], fx["config"])
    comp = mo.Computation.from_json(comp_j)
    ins = mo.make_inputs(comp, 2)
    (got,) = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64), want)


@pytest.mark.gpu
def test_tune_simcost_objective_and_seeding():
    """Objective::SimCost runs no kernel and returns the candidate with the
    lowest SimCost it visited (its objective equals mdh_b200_simcost of the
    returned config); SimCost seeding and a start configuration keep the
    history contract, and the start config is the first row."""
    from paper_2405_05118_b200 import mdh
    j = json.dumps(spec("matmul_fp32", [256, 256, 128]))
    best, hist, val = mdh.tune_ex(j, "B200", budget=8, seed=3, objective=mdh.OBJ_SIMCOST)
    rows = hist.strip().splitlines()
    assert rows[0] == "eval_index,config_hash,objective,valid" and len(rows) == 9
    assert val == mdh.simcost(j, "B200", best)[0]
    assert val == min(float(r.split(",")[2]) for r in rows[1:] if r.split(",")[3] == "1")
    # device-time objective, SimCost-seeded, starting from that best
    best2, hist2, secs = mdh.tune_ex(j, "B200", budget=6, seed=3, simcost_seeded=True, start_config=best)
    rows2 = hist2.strip().splitlines()
    assert len(rows2) == 7 and secs > 0
    # ties on the objective go to the lowest config hash (autotuner.cpp:263-271)
    best_hash = str(min(int(r.split(",")[1]) for r in rows[1:] if r.split(",")[3] == "1" and float(r.split(",")[2]) == val))
    assert rows2[1].split(",")[1] == best_hash  # the start configuration is evaluated first
    assert mdh.validate_config(j, "B200", best2) == ""
