"""CPU-side checks of the drop-in boundary (no GPU needed):
the C-ABI library loads, exports every entry point include/mdh_b200.h
declares, and its host front end (spec parser, md_hom rules, Table-1 config
validation) agrees with the unmodified reference."""
import ctypes
import json
import os
import re

import pytest

from conftest import REPO
from helpers import REFDATA, bundled, spec
from oracle import refbind


def header_symbols():
    text = open(os.path.join(REPO, "include", "mdh_b200.h")).read()
    return sorted(set(re.findall(r"\b(mdh_b200_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2405_05118_b200 import mdh
    lib = mdh.lib()
    declared = header_symbols()
    assert len(declared) >= 13
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(mdh.EXPORTED)


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(REPO, "paper_2405_05118_b200", "libmdh_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_sass_proves_blackwell_paths():
    import subprocess
    so = os.path.join(REPO, "paper_2405_05118_b200", "libmdh_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM", "IDP.4A"):
        assert mnemonic in sass, mnemonic


def _validate(spec_json, asm, cfg):
    from paper_2405_05118_b200 import mdh
    return mdh.validate_config(spec_json, asm, cfg)


@pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["matmul", "matvec", "mcc", "jacobi3d", "prl", "conv2d", "scan"])
@pytest.mark.parametrize("asm", ["CUDA", "CUDA+WRP", "OpenMP"])
def test_config_validation_agrees_with_reference(name, asm):
    text = json.dumps(bundled(name))
    for seed in range(6):
        for reduced in (True, False):
            cfg = refbind.sample_config(text, asm, seed, reduced=reduced, model_rules=False)
            want = refbind.validate(text, asm, cfg, model_rules=True)
            got = _validate(text, asm, cfg)
            assert (want == "") == (got == ""), (want, got)
            if want:
                assert want.split(":")[0] == got.split(":")[0]


@pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")
def test_published_fixtures_validate():
    for fx in ("tvm_gpu", "ppcg_gpu", "tvm_cpu", "pluto_cpu"):
        comp, cfg, asm = refbind.fixture(fx)
        assert refbind.validate(comp, asm, cfg) == ""
        assert _validate(comp, asm, cfg) == ""


def test_parse_errors_keep_reference_codes():
    from paper_2405_05118_b200 import mdh
    bad = bundled("matmul")
    bad["combine"] = ["cc", "cc", "pw:^"]
    with pytest.raises(mdh.MdhError) as e:
        mdh.validate_config(json.dumps(bad), "CUDA", "{}")
    assert e.value.code == "UnknownOperator"
    bad = bundled("matmul")
    bad["scalar"] = "out(1,1) = in(1,1) * ;"
    with pytest.raises(mdh.MdhError) as e:
        mdh.validate_config(json.dumps(bad), "CUDA", "{}")
    assert e.value.code == "ParseError"
    with pytest.raises(mdh.MdhError) as e:
        mdh.validate_config(json.dumps(bundled("matmul")), "NoSuchModel", "{}")
    assert e.value.code == "UnknownPreset"


def test_b200_model_rules():
    from paper_2405_05118_b200 import mdh
    s = json.dumps(spec("matmul_fp32", [256, 256, 64]))
    # 2048 CC parts on one CTA violates "Number of CCs limited"
    cfg = {"num_parts": [[1, 1, 1], [1, 1, 64], [1, 1, 1], [1, 1, 1], [1, 1, 1], [256, 256, 1]]}
    assert mdh.validate_config(s, "B200", json.dumps(cfg)).startswith("Number of CCs limited")
    cfg = {"num_parts": [[256, 256, 64], [1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1]]}
    assert mdh.validate_config(s, "B200", json.dumps(cfg)) == ""


def test_no_gpu_plan_creation_fails_loudly():
    """Without a device the product raises -- there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_05118_b200 import mdh
    with pytest.raises(mdh.MdhError) as e:
        mdh.Plan(spec("matvec_fp32", [8, 16]))
    assert e.value.code == "CudaError"
