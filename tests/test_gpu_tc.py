"""Tensor-core (tcgen05 kind::tf32) instance of the contraction family.

Exact mode (k/4 inputs, |k| <= 5) is representable in TF32 and every partial
sum is exact in FP32, so results must be bit-identical to the oracle.  In
U(-1,1) mode the bound is the stated TF32 one:
    |d_ij| <= 2^-9 * sum_k |a_ik| |b_kj|   (operand truncation to 10 bits + FP32 accumulate)
with sum|a||b| computed by the oracle itself on |A|, |B|."""
import numpy as np
import pytest

from helpers import exact_inputs, run_device, spec, uniform_inputs
from oracle import mdh_oracle as mo

CASES = [
    ("matmul_fp32", [128, 256, 64], "tc_gemm_tf32<256"),
    ("matmul_fp32", [256, 512, 96], "tc_gemm_tf32<256"),
    ("matmul_fp32", [128, 128, 32], "tc_gemm_tf32<128"),
    ("mcc_nhwc", [2, 8, 8, 64, 3, 3, 64], "tc_conv"),      # P padded 8 -> 16
    ("mcc_nhwc", [4, 16, 8, 64, 3, 3, 32], "tc_conv"),
    ("mcc_nhwc", [3, 20, 16, 64, 3, 3, 64], "tc_conv"),     # 2 p-blocks, ragged
    ("mcc_nhwc", [2, 16, 16, 64, 1, 1, 32], "tc_conv"),     # 1x1 taps
    # packed K-major operands (views no TMA box describes; K padded to 32)
    ("ccsdt_abcdef_gdab_efgc", [4, 4, 8, 8, 8, 4, 72], "tc_gemm_tf32<256"),
    ("ccsdt_abcdef_gdab_efgc", [8, 4, 4, 4, 8, 4, 40], "tc_gemm_tf32<128"),
]


def plan_tf32(j):
    from paper_2405_05118_b200 import mdh
    return mdh.Plan(j, math=mdh.MATH_TF32)


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,kernel", CASES)
def test_tf32_exact_mode_bit_identical(name, sizes, kernel):
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    plan = plan_tf32(j)
    d = plan.describe()
    kern = d["template"]["kernel"]
    # a 256-column tile may run as half of a 256 x 512 CTA-pair tile
    assert d["family"] == "contraction" and any(kern.startswith(kernel.replace("tc_gemm_tf32", v))
                                                for v in ("tc_gemm_tf32", "tc_gemm_pers", "tc_gemm_2sm")) or (
        kernel.endswith("<256") and kern.startswith("tc_gemm_2sm<512")), d
    assert d["family"] == "contraction" and d["template"].get("math") == "tf32", d
    ins = exact_inputs(comp, 4)
    (got,) = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64)[dfd], want[dfd])


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,kernel", CASES)
def test_tf32_uniform_mode_bound(name, sizes, kernel):
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    plan = plan_tf32(j)
    ins = uniform_inputs(comp, 8)
    (got,) = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    ((absw, _),) = mo.execute(comp, [np.abs(x) for x in ins])
    err = np.abs(got.astype(np.float64) - want)
    assert (err <= 2.0 ** -9 * absw + 1e-30)[dfd].all(), float((err / np.maximum(absw, 1e-30)).max())


@pytest.mark.gpu
def test_tf32_matmul_8192_exact_rows():
    import torch
    j = spec("matmul_fp32")
    comp = mo.Computation.from_json(j)
    plan = plan_tf32(j)
    assert "tc_gemm" in plan.describe()["template"]["kernel"]
    ins = exact_inputs(comp, 3)
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(x).to(t.dtype))
    (out,) = plan.empty(1)
    plan.run(d_in, [out])
    torch.cuda.synchronize()
    for lo in (0, 8191):
        ((part, dfd),), sh = mo.execute_box(comp, ins, {0: (lo, lo + 1)})
        assert np.array_equal(out[lo:lo + 1].cpu().numpy().astype(np.float64), part)


@pytest.mark.gpu
def test_tf32_mcc_full_image_exact():
    import torch
    j = spec("mcc_nhwc")
    comp = mo.Computation.from_json(j)
    plan = plan_tf32(j)
    assert "tc_conv" in plan.describe()["template"]["kernel"]
    ins = exact_inputs(comp, 3)
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(x).to(t.dtype))
    (out,) = plan.empty(1)
    plan.run(d_in, [out])
    torch.cuda.synchronize()
    ((part, dfd),), sh = mo.execute_box(comp, ins, {0: (255, 256)})
    assert np.array_equal(out[255:256].cpu().numpy().astype(np.float64), part)


@pytest.mark.gpu
def test_tf32_conv_matches_generic_tc_instance(monkeypatch):
    """The shifted-descriptor conv instance and the generic TMA-box instance
    (one box per tap) give the same bits on exact inputs."""
    j = spec("mcc_nhwc", [2, 16, 16, 64, 3, 3, 64])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 11)
    p1 = plan_tf32(j)
    assert p1.describe()["template"]["kernel"].startswith("tc_conv"), p1.describe()
    (a,) = run_device(p1, ins)
    monkeypatch.setenv("MDHB_TC_NO_CONV", "1")
    p2 = plan_tf32(j)
    assert p2.describe()["template"]["kernel"].startswith("tc_gemm"), p2.describe()
    (b,) = run_device(p2, ins)
    assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["MDHB_TC_NONPERSISTENT", "MDHB_TC_NO_TRANSPOSE", "MDHB_TC_1SM"])
def test_tf32_variants_agree(env, monkeypatch):
    """Non-persistent / MN-major instances give the same bits as the default."""
    j = spec("matmul_fp32", [256, 512, 96])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 6)
    (base,) = run_device(plan_tf32(j), ins)
    monkeypatch.setenv(env, "1")
    (var,) = run_device(plan_tf32(j), ins)
    assert np.array_equal(base, var)


@pytest.mark.gpu
def test_tf32_ccsdt_full_slices_exact():
    """Full CCSD(T) size on the tensor cores (packed operands) vs ++-slices."""
    import torch
    j = spec("ccsdt_abcdef_gdab_efgc")
    comp = mo.Computation.from_json(j)
    plan = plan_tf32(j)
    d = plan.describe()["template"]
    assert "tc_gemm" in d["kernel"] and "packed" in d["b_layout"], d
    ins = exact_inputs(comp, 3)
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(x).to(t.dtype))
    (out,) = plan.empty(1)
    plan.run(d_in, [out])
    torch.cuda.synchronize()
    for box in ({0: (0, 1), 1: (0, 2)}, {0: (23, 24), 3: (22, 24)}):
        ((part, dfd),), shifts = mo.execute_box(comp, ins, box)
        sl = tuple(slice(s, s + n) for s, n in zip(shifts[0], part.shape))
        assert np.array_equal(out[sl].cpu().numpy().astype(np.float64)[dfd], part[dfd]), box


@pytest.mark.gpu
@pytest.mark.parametrize("envs", [("MDHB_CONV_1SM",), ("MDHB_CONV_NOSW",), ("MDHB_CONV_1SM", "MDHB_CONV_NOSW"),
                                  ("MDHB_CONV_NO_TMA_STORE",), ("MDHB_CONV_1SM", "MDHB_CONV_NO_TMA_STORE")])
@pytest.mark.parametrize("sizes", [[3, 20, 16, 64, 3, 3, 64], [3, 56, 56, 64, 3, 3, 64]])
def test_tf32_conv_variants_bit_identical(envs, sizes, monkeypatch):
    """The single-CTA conv, the no-swizzle [c-group][p][q][4c] patch layout and
    the smem-transpose epilogue give the default instance's bits (CTA pair,
    128B-swizzled pixel-major patch, TMA-store epilogue); odd tile counts
    exercise the pair's ragged last tile, P = 20 / 56 the clipped p-blocks."""
    j = spec("mcc_nhwc", sizes)
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 12)
    (base,) = run_device(plan_tf32(j), ins)
    for e in envs:
        monkeypatch.setenv(e, "1")
    p = plan_tf32(j)
    (var,) = run_device(p, ins)
    assert np.array_equal(base, var), p.describe()


@pytest.mark.gpu
@pytest.mark.parametrize("envs", [("MDHB_CONV_2SM",), ("MDHB_CONV_NOSW",), ("MDHB_CONV_2SM", "MDHB_CONV_NOSW"),
                                  ("MDHB_CONV_NO_BF16F",), ("MDHB_CONV_BF16F_CFG=2,3,2",), ("MDHB_CONV_BF16F_CFG=3,2,2",),
                                  ("MDHB_CONV_BF16F_CFG=2,4,1",), ("MDHB_CONV_BF16F_CFG=4,2,1",)])
def test_bf16_conv_variants_bit_identical(envs, monkeypatch):
    """The bf16 conv instances (fused fp32 -> bf16 conversion with the default
    3 bf16 + 3 fp32 slots or the other slot / epilogue-buffer splits; separate
    conversion pass with CTA pair / single CTA, swizzled / plain patch) agree
    bit for bit."""
    from paper_2405_05118_b200 import mdh
    # C = 64: the fused instance is the default (C = 128 does not fit its rings)
    for sizes in ([3, 20, 16, 64, 3, 3, 64], [2, 56, 56, 64, 3, 3, 64]):
        j = spec("mcc_nhwc", sizes)
        comp = mo.Computation.from_json(j)
        ins = exact_inputs(comp, 13)
        monkeypatch.delenv("MDHB_CONV_2SM", raising=False)
        for e in envs:
            monkeypatch.delenv(e.partition("=")[0], raising=False)
        p0 = mdh.Plan(j, math=mdh.MATH_BF16)
        assert p0.describe()["template"]["kernel"].startswith("tc_conv_bf16f"), p0.describe()
        (base,) = run_device(p0, ins)
        ((part, dfd),), _ = mo.execute_box(comp, ins, {0: (0, 1)})  # image 0 against the oracle
        assert np.array_equal(base[:1].astype(np.float64)[dfd], part[dfd])
        for e in envs:
            k, _, v = e.partition("=")
            monkeypatch.setenv(k, v or "1")
        p = mdh.Plan(j, math=mdh.MATH_BF16)
        (var,) = run_device(p, ins)
        assert np.array_equal(base, var), p.describe()


BF16_CASES = [
    ("matmul_fp32", [256, 512, 96]),
    ("matmul_fp32", [512, 256, 200]),            # K padded to 256
    ("ccsdt_abcdef_gdab_efgc", [4, 4, 8, 8, 8, 4, 72]),
    ("mcc_nhwc", [2, 8, 8, 64, 3, 3, 64]),       # bf16 shifted-descriptor conv (tc_conv_bf16)
    ("mcc_nhwc", [3, 20, 16, 64, 3, 3, 128]),    # two 64-channel chunks, ragged p-blocks
]


def plan_bf16(j):
    from paper_2405_05118_b200 import mdh
    return mdh.Plan(j, math=mdh.MATH_BF16)


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes", BF16_CASES)
def test_bf16_exact_mode_bit_identical(name, sizes):
    """k/4 inputs are exact in bf16 and every partial sum is exact in the FP32
    accumulator: the BF16 tensor-core path is bit-identical to the oracle."""
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    plan = plan_bf16(j)
    d = plan.describe()
    assert d["family"] == "contraction" and d["template"]["math"] == "bf16", d
    ins = exact_inputs(comp, 4)
    (got,) = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64)[dfd], want[dfd])


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes", BF16_CASES)
def test_bf16_uniform_mode_bound(name, sizes):
    """|d_ij| <= 2^-8 * sum_k |a_ik| |b_kj| (operands rounded to 8 significant
    bits, FP32 accumulation) -- SURVEY 8(c)'s BF16 bound."""
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    plan = plan_bf16(j)
    ins = uniform_inputs(comp, 9)
    (got,) = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    ((absw, _),) = mo.execute(comp, [np.abs(x) for x in ins])
    err = np.abs(got.astype(np.float64) - want)
    assert (err <= 2.0 ** -8 * absw + 1e-30)[dfd].all(), float((err / np.maximum(absw, 1e-30)).max())


@pytest.mark.gpu
def test_bf16_matmul_8192_rows_exact():
    import torch
    j = spec("matmul_fp32")
    comp = mo.Computation.from_json(j)
    plan = plan_bf16(j)
    ins = exact_inputs(comp, 3)
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(x).to(t.dtype))
    (out,) = plan.empty(1)
    plan.run(d_in, [out])
    torch.cuda.synchronize()
    for lo in (0, 4097, 8191):
        ((part, dfd),), sh = mo.execute_box(comp, ins, {0: (lo, lo + 1)})
        assert np.array_equal(out[lo:lo + 1].cpu().numpy().astype(np.float64), part)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_conv_random_shapes_exact_all_maths(seed):
    """Seeded random NHWC convolution shapes (ragged P, Q in 8..64, channel
    counts that select or skip each conv instance) through FFMA, TF32 and BF16:
    exact-mode inputs give the oracle's values bit for bit on every path."""
    from paper_2405_05118_b200 import mdh
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 3))
    p = int(rng.integers(3, 40))
    q = 8 * int(rng.integers(1, 9))
    c = int(rng.choice([8, 16, 32, 64, 96, 128]))
    j = spec("mcc_nhwc", [n, p, q, 64, 3, 3, c])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, seed)
    ((want, dfd),) = mo.execute(comp, ins)
    for math in (mdh.MATH_FFMA, mdh.MATH_TF32, mdh.MATH_BF16):
        plan = mdh.Plan(j, math=math)
        (got,) = run_device(plan, ins)
        assert np.array_equal(got.astype(np.float64)[dfd], want[dfd]), (n, p, q, c, plan.describe()["template"])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_matmul_random_shapes_exact_all_maths(seed):
    """Seeded random MatMul shapes (tile-ragged M / N / K, including sizes no
    tensor-core or FFMA template takes and that fall to another instance):
    exact-mode inputs give the oracle's values bit for bit with every math."""
    from paper_2405_05118_b200 import mdh
    rng = np.random.default_rng(200 + seed)
    m, n, k = (int(rng.integers(1, 700)), int(rng.integers(1, 700)), int(rng.integers(1, 400)))
    j = spec("matmul_fp32", [m, n, k])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, seed)
    ((want, dfd),) = mo.execute(comp, ins)
    for math in (mdh.MATH_FFMA, mdh.MATH_TF32, mdh.MATH_BF16):
        plan = mdh.Plan(j, math=math)
        (got,) = run_device(plan, ins)
        assert np.array_equal(got.astype(np.float64)[dfd], want[dfd]), (m, n, k, plan.describe()["template"])


@pytest.mark.gpu
@pytest.mark.parametrize("math,kp", [(1, 72), (2, 80)])
def test_k_tail_step_exact(monkeypatch, math, kp):
    """K = 72 is not a multiple of the 128-byte k-tile: the packed operands
    keep K (TF32) or pad to 80 (BF16) and the last k-step lands 32-byte
    swizzled rows (SWIZZLE_32B TMA boxes, UMMA layout type 6)."""
    from paper_2405_05118_b200 import mdh
    monkeypatch.setenv("MDHB_TC_KTAIL", "1")
    j = spec("ccsdt_abcdef_gdab_efgc", [4, 4, 2, 8, 8, 24, 72])
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j, math=math)
    t = plan.describe()["template"]
    assert t["kernel"].startswith("tc_gemm_pers<192") and t.get("K_padded") == kp, t
    ins = exact_inputs(comp, 3)
    (got,) = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64)[dfd], want[dfd])
