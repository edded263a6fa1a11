"""The tuner's search space over Table-1 configurations (host only, no GPU):
every template instance of the stencil and the tensor-core GEMM families is
a canonical configuration the UNMODIFIED reference's validate accepts
(tuning.cpp:41-228 with the CUDA+WRP model rules), distinct per instance."""
import json

import pytest

from helpers import spec
from oracle import refbind

B200_ASM = '{"name": "B200", "mem": ["DM", "SM", "RM"], "core": ["SMX", "WRP", "CC"]}'


def space(name, sizes, family, **kw):
    from paper_2405_05118_b200 import mdh
    j = spec(name, sizes)
    return j, mdh.tune_space(j, family, **kw)


@pytest.mark.parametrize("sizes,n", [([512, 512, 512], 70), ([512, 32, 128], 50), ([64, 64, 256], 42)])
def test_stencil_space_every_divisor_times_every_schedule(sizes, n):
    # 5 schedules x every power-of-two TI dividing the i extent, plus the
    # LEAN schedule's 256- / 512-column tiles where they divide (j, k)
    j, sp = space("jacobi3d_fp32", sizes, "stencil")
    assert len(sp) == n and len({json.dumps(c, sort_keys=True) for c in sp}) == n
    tis = {sizes[0] // c["num_parts"][0][0] for c in sp}
    assert tis == {t for t in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512) if t <= sizes[0]}


def test_tc_space_covers_forms_tiles_groups_splits():
    from paper_2405_05118_b200 import mdh
    j, sp = space("matmul_fp32", [8192, 8192, 8192], "contraction", math=mdh.MATH_TF32)
    assert len(sp) >= 100
    rm_n = {c["num_parts"][5][1] for c in sp}        # RM parts of j = BN
    smx_k = {c["num_parts"][1][2] for c in sp}       # SMX parts of k = K split
    wrp_i = {c["num_parts"][2][0] for c in sp}       # WRP parts of i: 4 = 128-row tile, 8 = CTA pair
    assert rm_n == {64, 128, 256, 512} and smx_k == {1, 2, 4} and wrp_i == {4, 8}  # 512: CTA-pair 256 x 512
    _, small = space("matmul_fp32", [1024, 1024, 256], "contraction", math=mdh.MATH_TF32)
    assert len(small) >= 50


@pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,sizes,family,math", [("jacobi3d_fp32", [512, 32, 128], "stencil", 0),
                                                    ("matmul_fp32", [1024, 1024, 256], "contraction", 1),
                                                    ("matmul_fp32", [1024, 1024, 256], "contraction", 2),
                                                    ("matmul_fp32", [1024, 384, 128], "contraction", 1)])
def test_every_candidate_passes_the_reference_validate(name, sizes, family, math):
    from paper_2405_05118_b200 import mdh
    j, sp = space(name, sizes, family, math=math)
    text = json.dumps(j)
    for c in sp:
        assert mdh.validate_config(j, "B200", c) == ""
        assert refbind.validate(text, B200_ASM, json.dumps(c)) == ""
