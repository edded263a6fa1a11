"""SimCost (§8(f)4): the B200 library's restatement of the reference's
input-free cost model (simulate_trace + cost, interpreter.cpp:70-241;
simcost_objective, autotuner.cpp:58-62) must give the reference's value
exactly -- integer element counts times powers of two -- for reference-sampled
configurations of every bundled computation and for the published fixtures.
Host only: no GPU is touched."""
import json
import os

import pytest

from paper_2405_05118_b200 import cli, mdh
from oracle import refbind

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "simcost.json")))
DATA = os.path.join(HERE, "golden", "reference_data")


def _comp(name):
    with open(os.path.join(DATA, "computations", name)) as f:
        return f.read()


@pytest.mark.parametrize("case", GOLD["configs"], ids=lambda c: f'{c["computation"]}-{c["asm"]}-{c["seed"]}')
def test_simcost_matches_reference_golden(case):
    got, trace = mdh.simcost(_comp(case["computation"]), case["asm"], json.dumps(case["config"]))
    assert got == case["simcost"]
    assert trace["parallel_depth"] >= 3 and sum(trace["regions"].values()) > 0


@pytest.mark.parametrize("case", GOLD["fixtures"], ids=lambda c: c["fixture"])
def test_simcost_published_fixtures(case):
    name, spec, model, config = cli.load_fixture(case["fixture"], DATA)
    got, _ = mdh.simcost(spec, model, config)
    assert got == case["simcost"]


def test_simcost_rejects_invalid_config():
    text = _comp("matvec.json")
    cfg = json.loads(json.dumps(GOLD["configs"][[c["computation"] for c in GOLD["configs"]].index("matvec.json")]["config"]))
    cfg["num_parts"][0][0] = 3  # does not divide the dimension
    with pytest.raises(mdh.MdhError) as e:
        mdh.simcost(text, "CUDA+WRP", json.dumps(cfg))
    assert "InvalidConfig" in str(e.value) or "ParseError" in str(e.value)


def test_simcost_baseline_config():
    """NULL config = the baseline configuration (tuning.cpp:476-503)."""
    text = _comp("matmul.json")
    cost, trace = mdh.simcost(text, "CUDA+WRP")
    assert cost > 0 and set(trace["regions"]) <= {"DM", "SM", "RM"}


@pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("asm", ["CUDA+WRP", "CUDA", "OpenMP", "MultiGPU"])
def test_simcost_equals_unmodified_reference_live(asm):
    for f in sorted(os.listdir(os.path.join(DATA, "computations"))):
        text = _comp(f)
        for seed in range(3, 6):
            cfg = refbind.sample_config(text, asm, seed)
            assert mdh.simcost(text, asm, cfg)[0] == refbind.simcost(text, asm, cfg), (f, asm, seed)


@pytest.mark.parametrize("case", [c for c in GOLD["configs"] if "lowered" in c],
                         ids=lambda c: f'{c["computation"]}-{c["asm"]}')
def test_lowered_form_matches_reference_golden(case):
    """mdh_b200_lowered prints lower(e, m, cfg).pretty() byte for byte
    (lowering.cpp:185-222)."""
    assert mdh.lowered(_comp(case["computation"]), case["asm"], json.dumps(case["config"])) == case["lowered"]


@pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")
def test_lowered_form_equals_unmodified_reference_live():
    for f in sorted(os.listdir(os.path.join(DATA, "computations"))):
        text = _comp(f)
        for asm in ("CUDA", "MultiGPU"):
            cfg = refbind.sample_config(text, asm, 11)
            assert mdh.lowered(text, asm, cfg) == refbind.lowered(text, asm, cfg), (f, asm)
