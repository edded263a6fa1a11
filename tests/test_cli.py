"""The `mdh` driver (paper_2405_05118_b200/cli.py): subcommands,
output lines and exit codes of proj/tools/mdh_main.cpp."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

REFDATA = os.path.join(GOLDEN, "reference_data")


def run(args, capsys):
    from paper_2405_05118_b200 import cli
    rc = cli.main(args + (["--data", REFDATA] if args[0] != "examples" else ["--data", REFDATA]))
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_exit_codes_mirror_the_reference():
    from paper_2405_05118_b200 import cli
    assert cli.exit_code_for("ParseError") == 3
    for c in ("InvalidConfig", "Mismatch", "NoValidConfigFound", "NonDivisible", "MixedIncompatibleOperators",
              "UnknownPreset", "UnknownFixture"):
        assert cli.exit_code_for(c) == 2
    assert cli.exit_code_for("CudaError") == 1


def test_missing_spec_is_a_parse_error(capsys):
    rc, _, err = run(["verify", "--spec", "no_such_computation"], capsys)
    assert rc == 3 and "ParseError" in err


def test_unknown_fixture(capsys):
    rc, _, err = run(["verify", "--fixture", "no_such_fixture"], capsys)
    assert rc == 2 and "UnknownFixture" in err


def test_bad_arguments_exit_3():
    from paper_2405_05118_b200 import cli
    assert cli.main(["frobnicate"]) == 3


def test_examples_lists_bundled_computations(capsys):
    rc, out, _ = run(["examples"], capsys)
    assert rc == 0
    assert "matvec: dims" in out and "fixture tvm_gpu: matmul_resnet on CUDA" in out


def test_driver_inputs_follow_the_reference_rng():
    """mdh_main.cpp:46-66: mt19937_64(seed ^ 0x9e3779b97f4a7c15), below(11) - 5."""
    from paper_2405_05118_b200 import cli
    g = cli._MT64(5489)
    for _ in range(9999):
        g.next()
    assert g.next() == 9981545732273789042   # the C++ standard's check value


@pytest.mark.gpu
@pytest.mark.parametrize("spec", ["matvec", "matmul", "mcc", "jacobi3d", "histo", "scan", "prl"])
def test_verify_bundled(spec, capsys):
    rc, out, _ = run(["verify", "--spec", spec], capsys)
    assert rc == 0 and "1/1 configurations pass" in out, out


@pytest.mark.gpu
def test_verify_published_fixture(capsys):
    """tvm_gpu: TVM's MatMul decomposition (the reference's AC4 fixture)."""
    rc, out, _ = run(["verify", "--fixture", "tvm_gpu"], capsys)
    assert rc == 0 and "config tvm_gpu: pass" in out, out


@pytest.mark.gpu
@pytest.mark.parametrize("spec", ["matvec", "jacobi3d", "mcc", "prl"])
def test_verify_random_configurations(spec, capsys):
    """`verify --random 3`: three sampled configurations (random prime-factor
    placements over the layers), each executed -- on a specialised template
    when it can instantiate the sample, else on the emitted / VM kernels --
    and checked against the device reference executor."""
    rc, out, _ = run(["verify", "--spec", spec, "--random", "3", "--seed", "7"], capsys)
    assert rc == 0 and out.count(": pass (hash=") == 3 and "3/3 configurations pass" in out, out
    assert "config random:0" in out and "config random:2" in out


@pytest.mark.gpu
def test_verify_invalid_config_exit_2(tmp_path, capsys):
    cfg = tmp_path / "bad.json"
    cfg.write_text(json.dumps({"num_parts": [[3, 1]]}))
    rc, out, err = run(["verify", "--spec", "matvec", "--config", str(cfg)], capsys)
    assert rc in (2, 3), (out, err)


@pytest.mark.gpu
def test_emit_prints_the_nvrtc_kernel(capsys):
    rc, out, _ = run(["emit", "--spec", "histo"], capsys)
    assert rc == 0 and 'extern "C" __global__' in out and "mdh_emitted" in out


@pytest.mark.gpu
@pytest.mark.parametrize("spec", ["histo", "matvec", "scan"])
def test_emit_gate_compile_runs_the_kernel(spec, capsys):
    """`emit --gate-compile` (mdh_main.cpp:180-205): the compiled kernel is
    run on the driver's inputs and checked against the device reference."""
    rc, out, err = run(["emit", "--spec", spec, "--gate-compile", "--f64"], capsys)
    assert rc == 0 and "gate passed" in err, err


@pytest.mark.gpu
@pytest.mark.parametrize("objective", [None, "compiled"])  # None: the reference's default, simcost
def test_tune_writes_history_with_reference_columns(objective, tmp_path, capsys):
    hist = tmp_path / "h.csv"
    best = tmp_path / "best.json"
    extra = ["--objective", objective] if objective else []
    rc, out, _ = run(["tune", "--spec", "matvec", "--budget", "3", "--history", str(hist), "--out", str(best)] + extra,
                     capsys)
    assert rc == 0 and "evaluations: 3" in out
    rows = hist.read_text().strip().splitlines()
    assert rows[0] == "eval_index,config_hash,objective,valid" and len(rows) == 4
    assert "num_parts" in json.loads(best.read_text())


@pytest.mark.gpu
def test_tune_simcost_from_published_fixture(tmp_path, capsys):
    """`tune --objective simcost --seed-simcost --start tvm_gpu`: the fixture's
    configuration is the first history row and the best objective is the
    SimCost of the written configuration."""
    from paper_2405_05118_b200 import cli, mdh
    hist = tmp_path / "h.csv"
    best = tmp_path / "best.json"
    rc, out, _ = run(["tune", "--spec", "matmul_resnet", "--asm", "CUDA", "--objective", "simcost", "--seed-simcost",
                      "--start", "tvm_gpu", "--budget", "6", "--history", str(hist), "--out", str(best)], capsys)
    assert rc == 0 and "evaluations: 6" in out, out
    rows = hist.read_text().strip().splitlines()
    assert len(rows) == 7
    _, spec, model, cfg = cli.load_fixture("tvm_gpu")
    start_cost, _ = mdh.simcost(cli.load_spec("matmul_resnet"), "CUDA", cfg)
    assert float(rows[1].split(",")[2]) == start_cost
    best_obj = float([l for l in out.splitlines() if l.startswith("best objective:")][0].split(":")[1])
    assert abs(best_obj - mdh.simcost(cli.load_spec("matmul_resnet"), "CUDA", best.read_text())[0]) <= 1e-6 * best_obj


@pytest.mark.gpu
def test_run_reproduces_a_frozen_reference_vector(tmp_path, capsys):
    ref = os.path.join(REFDATA, "refs", "matmul.ref.json")
    out_file = tmp_path / "o.json"
    rc, _, _ = run(["run", "--spec", "matmul", "--inputs", ref, "--out", str(out_file)], capsys)
    assert rc == 0
    got = json.loads(out_file.read_text())["outputs"]
    want = json.load(open(ref))["outputs"]
    for name, g in want.items():
        w = np.array([0 if x is None else x for x in g["data"]], dtype=np.float64)
        assert np.array_equal(np.array(got[name]["data"], dtype=np.float64), w), name


def test_lower_prints_the_reference_lowered_form(tmp_path, capsys):
    """`lower --fixture tvm_gpu`: the reference's pretty form of the published
    TVM configuration (host only; golden text from the unmodified reference
    when oracle/_ref is built)."""
    rc, out, _ = run(["lower", "--fixture", "tvm_gpu"], capsys)
    assert rc == 0 and out.startswith("lowered computation=matmul_resnet model=CUDA\n"), out[:200]
    assert out.splitlines()[1] == "de level=(-) tag=(-) op=iv" and out.rstrip().endswith("re level=(-) tag=(-) op=ov")
    from oracle import refbind
    if refbind.available():
        from paper_2405_05118_b200 import cli
        comp, cfg, asm = refbind.fixture("tvm_gpu")
        assert out == refbind.lowered(comp, asm, cfg)
