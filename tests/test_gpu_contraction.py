"""Contraction family (MatVec, MatMul, ResNet-50 FC, MCC NHWC, CCSD(T)) vs the
oracle.  Exact mode (the reference's own k/4 inputs, support.hpp:41-45) must be
bit-identical; U(-1,1) inputs must satisfy |d| <= 1e-5 sqrt(K) max(|ref|,1)."""
import numpy as np
import pytest

from helpers import assert_close, exact_inputs, run_device, spec, uniform_inputs
from oracle import mdh_oracle as mo

SMALL = [
    ("matvec_fp32", [64, 128], "gemv"),
    ("matvec_fp32", [300, 256], "gemv"),
    ("matmul_fp32", [128, 128, 64], "sgemm"),
    ("matmul_fp32", [256, 192, 72], "sgemm"),
    ("matmul_fp32", [64, 64, 8], "sgemm"),
    ("matmul_fp32", [256, 2048, 96], "sgemm_pipe<128x128,V16,V16"),   # A transposed by the layout pass; short K: 128 x 128
    ("matmul_fp32", [384, 2048, 40], "sgemm_pipe<128x128,V16,V16"),   # K = 32 + a partial k-tile of 8
    ("matmul_fp32", [256, 1024, 520], "sgemm_pipe<128x64,V16,V16"),   # long K: 128 x 64, 32 x 16 + 8
    ("mcc_nhwc", [2, 8, 8, 64, 3, 3, 64], "sgemm_pipe<128x64"),   # implicit GEMM (FFMA2)
    ("mcc_nhwc", [4, 8, 16, 64, 3, 3, 16], ""),                   # short K: patch-reuse conv or GEMM
    ("mcc_nhwc", [3, 10, 16, 64, 3, 3, 24], "ffma_conv"),      # no 128-row tiling of N x P x Q: patch-reuse conv
    ("mcc_nhwc", [2, 56, 56, 64, 3, 3, 64], "sgemm_pipe<128x64"),  # conv2_x images
    ("ccsdt_abcdef_gdab_efgc", [4, 4, 4, 4, 4, 4, 8], "sgemm"),
    ("ccsdt_abcdef_gdab_efgc", [8, 4, 4, 4, 8, 4, 16], "sgemm"),
    ("matmul_resnet_fc", [16, 1000, 2048], "skinny_cluster<16>"),
    ("matmul_resnet_fc", [1, 1000, 2048], "skinny_cluster<16>"),    # inference shape (M = 1)
    ("matmul_resnet_fc", [5, 36, 512], "skinny_cluster<16>"),       # ragged N strip, cluster of 8
    ("matmul_resnet_fc", [24, 100, 256], "skinny_cluster<32>"),     # 17..32 rows, cluster of 4
    ("matmul_resnet_fc", [32, 64, 128], "skinny_cluster<32>"),      # cluster of 2
    ("matmul_resnet_fc", [16, 100, 328], "skinny_partial"),         # K not a multiple of 128: v1
]


def K_of(comp):
    return int(np.prod([n for n, (k, _) in zip(comp.sizes, comp.combine) if k == "pw"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,kernel", SMALL)
def test_exact_mode_bit_identical(name, sizes, kernel):
    from paper_2405_05118_b200 import mdh
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j)
    d = plan.describe()
    if kernel:
        assert d["family"] == "contraction" and kernel in d["template"]["kernel"], d
    ins = exact_inputs(comp, 5)
    got = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got[0].astype(np.float64)[dfd], want[dfd])


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,kernel", SMALL)
def test_uniform_mode_within_tolerance(name, sizes, kernel):
    from paper_2405_05118_b200 import mdh
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j)
    ins = uniform_inputs(comp, 2)
    got = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert_close(got[0], want, dfd, K_of(comp), name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["matmul", "matmul_t", "bmatmul", "conv2d", "mcc", "dot", "matvec"])
def test_bundled_contractions_vs_oracle(name):
    """Bundled reference specs (i64) at sizes the tile menu accepts or not --
    every one must run on the device and agree exactly."""
    from helpers import bundled
    from paper_2405_05118_b200 import mdh
    sizes = {"matmul": [64, 64, 16], "matmul_t": [64, 128, 24], "bmatmul": [3, 6, 6, 6], "conv2d": [8, 8, 3, 3],
             "mcc": [2, 4, 4, 2, 3, 3, 2], "dot": [1000], "matvec": [64, 128]}[name]
    j = bundled(name, sizes)
    for t in j["inputs"] + j["outputs"]:
        t["type"] = "f64"
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j)
    ins = exact_inputs(comp, 9)
    got = run_device(plan, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got[0].astype(np.float64)[dfd], want[dfd]), plan.describe()


def _full(name, slices):
    """Full BASELINE size on the device; oracle on ++-slices of dim 0."""
    import torch
    from paper_2405_05118_b200 import mdh
    j = spec(name)
    comp = mo.Computation.from_json(j)
    plan = mdh.Plan(j)
    d = plan.describe()
    assert d["family"] == "contraction", d
    ins = exact_inputs(comp, 3)
    d_in = plan.empty(0)
    for t, x in zip(d_in, ins):
        t.copy_(torch.from_numpy(x).to(t.dtype))
    (out,) = plan.empty(1)
    plan.run(d_in, [out])
    torch.cuda.synchronize()
    for box in slices:
        if isinstance(box, tuple):
            box = {0: box}
        ((part, dfd),), shifts = mo.execute_box(comp, ins, box)
        sl = tuple(slice(s, s + n) for s, n in zip(shifts[0], part.shape))
        got = out[sl].cpu().numpy().astype(np.float64)
        assert np.array_equal(got[dfd], part[dfd]), (name, box)


@pytest.mark.gpu
def test_mcc_ffma_conv_matches_implicit_gemm(monkeypatch):
    """The patch-reuse conv instance and the table-driven implicit GEMM (the
    default where it tiles) agree bit for bit on exact inputs (and with the
    oracle)."""
    from paper_2405_05118_b200 import mdh
    j = spec("mcc_nhwc", [2, 8, 8, 64, 3, 3, 64])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 9)
    monkeypatch.setenv("MDHB_FFMA_CONV", "1")
    p = mdh.Plan(j)
    assert "ffma_conv" in p.describe()["template"]["kernel"]
    (a,) = run_device(p, ins)
    monkeypatch.delenv("MDHB_FFMA_CONV")
    q = mdh.Plan(j)
    assert "sgemm" in q.describe()["template"]["kernel"]
    (b,) = run_device(q, ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(a, b) and np.array_equal(a.astype(np.float64)[dfd], want[dfd])


@pytest.mark.gpu
@pytest.mark.parametrize("sizes", [[2, 8, 8, 64, 3, 3, 64], [1, 16, 8, 64, 1, 1, 40]])
def test_mcc_k_contiguous_a_tile_bit_identical(monkeypatch, sizes):
    """The K-contiguous A tile (sgemm_pipe_ak, opt-in) and the S4 form of the
    implicit GEMM agree bit for bit on U(-1,1) inputs and match the oracle on
    exact ones; the 1 x 1 filter over C = 40 gives K = 40 = 2 x 16 + 8, the
    partial last k-tile."""
    from paper_2405_05118_b200 import mdh
    j = spec("mcc_nhwc", sizes)
    comp = mo.Computation.from_json(j)
    for ins in (exact_inputs(comp, 9), uniform_inputs(comp, 5)):
        p = mdh.Plan(j)
        if "sgemm_pipe" not in p.describe()["template"]["kernel"]:
            pytest.skip(p.describe()["template"]["kernel"])
        (a,) = run_device(p, ins)
        monkeypatch.setenv("MDHB_PIPE_AK", "1")
        q = mdh.Plan(j)
        assert "K16" in q.describe()["template"]["kernel"]
        (b,) = run_device(q, ins)
        monkeypatch.delenv("MDHB_PIPE_AK")
        assert np.array_equal(a, b)
    ((want, dfd),) = mo.execute(comp, exact_inputs(comp, 9))
    monkeypatch.setenv("MDHB_PIPE_AK", "1")  # read at launch
    (c,) = run_device(q, exact_inputs(comp, 9))
    assert np.array_equal(c.astype(np.float64)[dfd], want[dfd])


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["MDHB_SKINNY_TABLES", "MDHB_SKINNY_TMA", "MDHB_SKINNY_TXFOLD"])
@pytest.mark.parametrize("sizes", [[16, 1000, 2048], [5, 36, 512], [1, 1000, 2048], [24, 100, 256]])
def test_fc_variants_bit_identical(monkeypatch, sizes, env):
    """skinny_cluster computes affine row / column offsets in the kernel and
    loads B by cp.async; with MDHB_SKINNY_TABLES=1 it reads the plan's tables,
    with MDHB_SKINNY_TMA=1 it loads the B slice by TMA tensor copies (zero
    fill past N), with MDHB_SKINNY_TXFOLD=1 the slices meet by st.async pushes
    on per-owner mbarriers: all bit-identical on U(-1,1) inputs, and exact
    against the oracle on exact ones."""
    from paper_2405_05118_b200 import mdh
    j = spec("matmul_resnet_fc", sizes)
    comp = mo.Computation.from_json(j)
    ins = uniform_inputs(comp, 4)
    (a,) = run_device(mdh.Plan(j), ins)
    monkeypatch.setenv(env, "1")
    q = mdh.Plan(j)
    assert "skinny_cluster" in q.describe()["template"]["kernel"]
    (b,) = run_device(q, ins)
    assert np.array_equal(a, b)
    ex = exact_inputs(comp, 6)
    ((want, dfd),) = mo.execute(comp, ex)
    (c,) = run_device(q, ex)
    assert np.array_equal(c.astype(np.float64)[dfd], want[dfd])


@pytest.mark.gpu
def test_matvec_full_size_exact():
    _full("matvec_fp32", [(0, 4096)])


@pytest.mark.gpu
def test_matmul_8192_rows_exact():
    _full("matmul_fp32", [(0, 1), (8191, 8192)])


@pytest.mark.gpu
def test_mcc_full_images_exact():
    _full("mcc_nhwc", [(0, 1), (255, 256)])


@pytest.mark.gpu
def test_ccsdt_full_slices_exact():
    _full("ccsdt_abcdef_gdab_efgc", [{0: (0, 1), 1: (0, 2)}, {0: (23, 24), 3: (22, 24)}])


@pytest.mark.gpu
def test_fc_full_exact():
    _full("matmul_resnet_fc", [(0, 16)])
