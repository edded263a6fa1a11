"""The reference-side binding, compiled (integration/b200_adaptor.*, built
by `make -C oracle adaptor` against the unmodified reference headers and
linked with the reference library + libmdh_b200.so):

  * reference_execute(e, in) == mdh::b200::execute(e, in), cell for cell and
    definedness for definedness, on every bundled computation and the
    BASELINE specs (f64 storage: bit-identical; FP32 storage on the
    reference's exact inputs: identical too);
  * the configuration-ordered form b200::execute(e, m, cfg, in) under
    configurations the reference itself samples;
  * the reference's OWN hill_climb / tune loop driving the device objective
    (b200::time_evaluator / b200::tune, the EvaluateFn binding)."""
import ctypes
import json
import os

import pytest

from conftest import GOLDEN, REPO
from oracle import refbind

SO = os.path.join(REPO, "oracle", "_ref", "libmdh_b200_adaptor.so")
needs = pytest.mark.skipif(not os.path.exists(SO), reason="adaptor not built (needs /root/reference at build time)")
COMPS = os.path.join(GOLDEN, "reference_data", "computations")
SMALL_SPECS = {"matvec_fp32": [16, 32], "jacobi3d_fp32": [8, 8, 8], "matmul_fp32": [8, 8, 16],
               "matmul_resnet_fc": [4, 40, 64], "mcc_nhwc": [2, 6, 6, 8, 3, 3, 8],
               "ccsdt_abcdef_gdab_efgc": [3, 3, 3, 3, 3, 3, 8], "prl_max": [64, 4096], "scan_i32": [100]}


def lib():
    L = ctypes.CDLL(SO)
    L.adaptor_last_error.restype = ctypes.c_char_p
    L.adaptor_check_execute.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
    L.adaptor_hill_climb.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64,
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_int)]
    L.adaptor_tune.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_char_p,
                               ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]
    return L


def check(L, comp, asm=b"", cfg=b"", seed=1, f64=1, math=0):
    bad = ctypes.c_int64(-2)
    rc = L.adaptor_check_execute(comp, asm, cfg, seed, f64, math, ctypes.byref(bad))
    assert rc == 0, L.adaptor_last_error().decode()
    return bad.value


def all_specs():
    out = []
    for f in sorted(os.listdir(COMPS)):
        with open(os.path.join(COMPS, f)) as fh:
            out.append((f[:-5], fh.read()))
    for n, sz in SMALL_SPECS.items():
        with open(os.path.join(REPO, "specs", n + ".json")) as fh:
            j = json.load(fh)
        j["sizes"] = sz
        out.append((n, json.dumps(j)))
    return out


def dyadic_literals(scalar):
    import re
    for lit in re.findall(r"\d+\.\d+(?:[eE][-+]?\d+)?", scalar):
        if float(lit) * 256 != int(float(lit) * 256):
            return False
    return True


@needs
def test_adaptor_exports():
    L = lib()
    for s in ("adaptor_check_execute", "adaptor_hill_climb", "adaptor_tune", "adaptor_last_error"):
        assert hasattr(L, s)


@needs
@pytest.mark.gpu
@pytest.mark.parametrize("name,text", all_specs(), ids=[n for n, _ in all_specs()])
def test_reference_execute_equals_b200_execute(name, text):
    L = lib()
    if json.loads(text)["sizes"] and max(json.loads(text)["sizes"]) > 1024 and name == "matmul_resnet":
        j = json.loads(text)
        j["sizes"] = [4, 40, 64]
        text = json.dumps(j)
    assert check(L, text.encode(), f64=1) == 0            # f64 storage: bit-identical
    if dyadic_literals(json.loads(text)["scalar"]):       # Jacobi's 0.4 / 0.1 are not exact in FP32
        assert check(L, text.encode(), seed=3, f64=0) == 0  # FP32 storage on the reference's exact inputs


@needs
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["matvec", "matmul", "mcc", "jacobi3d", "prl", "scan", "histo", "bmatmul"])
def test_configured_execute_equals_reference(name):
    L = lib()
    with open(os.path.join(COMPS, name + ".json")) as f:
        text = f.read()
    for seed in range(3):
        cfg = refbind.sample_config(text, "CUDA+WRP", seed) if refbind.available() else ""
        assert check(L, text.encode(), b"CUDA+WRP", cfg.encode(), seed=seed + 5) == 0


@needs
@pytest.mark.gpu
def test_reference_hill_climb_with_device_objective():
    L = lib()
    with open(os.path.join(REPO, "specs", "matvec_fp32.json")) as f:
        j = json.load(f)
    j["sizes"] = [256, 512]
    s0, s1, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    rc = L.adaptor_hill_climb(json.dumps(j).encode(), b"CUDA+WRP", 4, 7, ctypes.byref(s0), ctypes.byref(s1), ctypes.byref(n))
    assert rc == 0, L.adaptor_last_error().decode()
    assert 0 < s1.value <= s0.value < 1.0 and 1 <= n.value <= 4


@needs
@pytest.mark.gpu
def test_b200_tune_through_the_reference_search():
    L = lib()
    with open(os.path.join(REPO, "specs", "matvec_fp32.json")) as f:
        j = json.load(f)
    j["sizes"] = [256, 512]
    best = ctypes.create_string_buffer(1 << 20)
    csv = ctypes.create_string_buffer(1 << 16)
    obj = ctypes.c_double()
    rc = L.adaptor_tune(json.dumps(j).encode(), b"CUDA+WRP", 6, 3, best, 1 << 20, csv, 1 << 16, ctypes.byref(obj))
    assert rc == 0, L.adaptor_last_error().decode()
    rows = csv.value.decode().strip().splitlines()
    assert rows[0] == "eval_index,config_hash,objective,valid" and len(rows) == 7
    assert 0 < obj.value < 1.0 and json.loads(best.value.decode())["num_parts"]
