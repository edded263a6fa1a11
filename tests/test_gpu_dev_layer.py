"""The multi-GPU DEV layer through the C ABI, on the CUDA
kernels.  The pool gives one GPU per run, so G shards share cuda:0 here
(device_ids [0]*G): ++ splits run G shard kernels on their slabs with no
communication; point-wise splits combine through the peer-memory combine
kernel (the NCCL all-reduce path needs distinct devices and is exercised
only on a multi-GPU node -- unmeasured here).  Every recombined result must
equal the unsplit oracle / the unsplit device plan bit for bit."""
import json
import os
import socket

import numpy as np
import pytest

from conftest import REPO
from helpers import exact_inputs, run_device, spec, uniform_inputs
from oracle import mdh_oracle as mo


def mplan(j, G, **kw):
    from paper_2405_05118_b200 import mdh
    return mdh.MultiPlan(j, G, device_ids=[0] * G, **kw)


def prl_inputs(nq, nr, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 3, (nq, 4)).astype(np.int64), rng.integers(0, 3, (nr, 4)).astype(np.int64),
            np.array([3, 5, 7, 9], dtype=np.int64)]


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4])
def test_matvec_row_split_no_communication(G):
    j = spec("matvec_fp32", [1024, 2048])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 1)
    mp = mplan(j, G)
    d = mp.describe()
    assert d["split_dim"] == 1 and d["split_kind"] == "cc" and d["combine"] == "none", d
    (got,) = mp.run_host(ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64), want)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4])
def test_matvec_k_split_combines_with_sum(G):
    j = spec("matvec_fp32", [512, 4096])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 2)
    mp = mplan(j, G, split_dim=2)
    d = mp.describe()
    assert d["split_kind"] == "pw" and d["combine"] == "peer", d
    (got,) = mp.run_host(ins)
    ((want, _),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64), want)  # exact mode: the sum order cannot show


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
def test_prl_record_split_max_of_packed_keys(G):
    nq, nr = 512, 65536
    j = spec("prl_max", [nq, nr])
    ins = prl_inputs(nq, nr, G)
    from paper_2405_05118_b200 import mdh
    mp = mplan(j, G, split_dim=2, int_storage=mdh.I32)
    d = mp.describe()
    assert d["split_kind"] == "pw" and all(s["plan"]["family"] == "prl" for s in d["shards"]), d
    (got,) = mp.run_host(ins)
    ((want, _),) = mo.execute(mo.Computation.from_json(j), ins)
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4])
def test_prl_record_split_custom_max_prl(G):
    nq, nr = 256, 32768
    with open(os.path.join(REPO, "specs", "extensions", "prl_max_prl.json")) as f:
        j = json.load(f)
    j["sizes"] = [nq, nr]
    ins = prl_inputs(nq, nr, 7 + G)
    w, r = mplan(j, G, split_dim=2).run_host(ins)
    ((best, _),) = mo.execute(mo.Computation.from_json(spec("prl_max", [nq, nr])), ins)
    assert np.array_equal(w, best >> 20) and np.array_equal(r, (1 << 20) - 1 - (best & ((1 << 20) - 1)))


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
def test_prl_query_split(G):
    nq, nr = 2048, 16384
    j = spec("prl_max", [nq, nr])
    ins = prl_inputs(nq, nr, 3)
    mp = mplan(j, G)
    assert mp.describe()["split_kind"] == "cc"
    (got,) = mp.run_host(ins)
    ((want, _),) = mo.execute(mo.Computation.from_json(j), ins)
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
def test_jacobi3d_z_slabs_equal_unsplit_plan(G):
    from paper_2405_05118_b200 import mdh
    j = spec("jacobi3d_fp32", [64, 64, 256])
    comp = mo.Computation.from_json(j)
    ins = uniform_inputs(comp, 5)
    (whole,) = mdh.Plan(j).run_host(ins)
    mp = mplan(j, G)
    d = mp.describe()
    assert d["split_dim"] == 1 and all(s["plan"]["family"] == "stencil" for s in d["shards"]), d
    assert [s["range"] for s in d["shards"]] == [[64 // G * g, 64 // G * (g + 1)] for g in range(G)]
    (got,) = mp.run_host(ins)
    assert np.array_equal(got, whole)  # same kernel, same arithmetic per point


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,dim", [("mcc_nhwc", [4, 12, 16, 64, 3, 3, 32], 1),
                                            ("mcc_nhwc", [2, 16, 16, 64, 3, 3, 32], 2),
                                            ("ccsdt_abcdef_gdab_efgc", [8, 4, 4, 4, 8, 4, 40], 1),
                                            ("matmul_fp32", [256, 384, 128], 1),
                                            ("matmul_fp32", [256, 384, 128], 3)])
def test_contractions_split_exact(name, sizes, dim):
    j = spec(name, sizes)
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 4)
    (got,) = mplan(j, 2, split_dim=dim).run_host(ins)
    ((want, dfd),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64)[dfd], want[dfd])


def jacobi_np(v, sweeps):
    v = v.astype(np.float32).copy()
    for _ in range(sweeps):
        c = v[1:-1, 1:-1, 1:-1]
        w = (np.float32(0.4) * c + np.float32(0.1) * (v[:-2, 1:-1, 1:-1] + v[2:, 1:-1, 1:-1] + v[1:-1, :-2, 1:-1] +
                                                   v[1:-1, 2:, 1:-1] + v[1:-1, 1:-1, :-2] + v[1:-1, 1:-1, 2:]))
        v[1:-1, 1:-1, 1:-1] = w
    return v


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4])
def test_iterated_jacobi_with_halo_exchange(G):
    """Iterated sweeps: ghost planes exchanged between neighbouring shards
    after every sweep.  The G-shard state after 5 sweeps equals the 1-shard
    state bit for bit, and the plain numpy iteration within tolerance."""
    import torch
    j = spec("jacobi3d_fp32", [32, 32, 128])
    comp = mo.Computation.from_json(j)
    (v0,) = uniform_inputs(comp, 6)
    states = {}
    for g in (1, G):
        mp = mplan(j, g)
        dv = mp.empty(0)
        dw = mp.empty(1)
        for s in range(g):
            dv[s][0].copy_(torch.from_numpy(np.ascontiguousarray(mp.slab(s, 0, 0, v0))).float())
        mp.iterate(dv, dw, 5)
        torch.cuda.synchronize()
        out = v0.astype(np.float32).copy()
        for s in range(g):
            st = mp.inputs[s][0]["start"]
            n = mp.inputs[s][0]["shape"][0]
            out[st + 1:st + n - 1] = dv[s][0].cpu().numpy()[1:n - 1]
        states[g] = out
    assert np.array_equal(states[1], states[G])
    want = jacobi_np(v0, 5)
    assert np.abs(states[G] - want).max() <= 1e-5 * 3


@pytest.mark.gpu
def test_mplan_time_is_max_over_shards():
    j = spec("jacobi3d_fp32", [128, 128, 256])
    mp = mplan(j, 2)
    d_in, d_out = mp.empty(0), mp.empty(1)
    for row in d_in:
        for t in row:
            t.uniform_(-1, 1)
    t = mp.time(d_in, d_out, warmup=2, reps=5)
    assert 0 < t < 0.1


# ---- one process per GPU: rank plans under torch.distributed -------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, name, sizes, split_dim, q):
    """Each rank: its shard's plan (the CUDA kernels on cuda:0), the
    point-wise combine over the process group (gloo here, on host copies; the
    NCCL path is the same call with an NCCL id), ++ slabs gathered."""
    import sys
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist
    from paper_2405_05118_b200 import mdh
    from paper_2405_05118_b200.shard import combine_op
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        with open(os.path.join(REPO, "specs", name + ".json")) as f:
            j = json.load(f)
        j["sizes"] = sizes
        comp = mo.Computation.from_json(j)
        rng = np.random.default_rng(1)
        ins = ([rng.integers(0, 3, s).astype(np.int64) for s in mo.input_shapes(comp)[:2]] +
               [np.array([3, 5, 7, 9], np.int64)]) if name == "prl_max" else mo.make_inputs(comp, 1)
        p = mdh.rank_plan(j, world, rank, device=0, split_dim=split_dim)
        sh = p.describe()["template"]["shard"]
        mine = []
        for x, (r, st), info in zip(ins, sh["in"], p.inputs):
            if r < 0:
                mine.append(x)
            else:
                idx = [slice(None)] * x.ndim
                idx[r] = slice(st, st + info["shape"][r])
                mine.append(x[tuple(idx)])
        outs = run_device(p, mine)
        res = []
        for o, (r, st) in zip(outs, sh["out"]):
            t = torch.from_numpy(np.ascontiguousarray(o))
            if sh["split_kind"] == "pw":
                op = j["combine"][sh["split_dim"] - 1].split(":")[1]
                dist.all_reduce(t, op=combine_op(dist, op))
                res.append(t.numpy())
            else:
                parts = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                res.append(torch.cat(parts, dim=r).numpy())
        if rank == 0:
            want = mo.execute(comp, ins)
            q.put(all(np.array_equal(g.astype(np.float64) if g.dtype.kind == "f" else g, w[0]) for g, w in zip(res, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name,sizes,split_dim", [("prl_max", [256, 8192], 2), ("prl_max", [256, 8192], 1),
                                                  ("matvec_fp32", [512, 1024], 2), ("matvec_fp32", [512, 1024], 1)])
def test_world2_rank_plans_run_the_kernels(name, sizes, split_dim):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, name, sizes, split_dim, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(60)
    assert ok and all(p.exitcode == 0 for p in procs)


@pytest.mark.gpu
def test_rank_plan_nccl_allreduce_runs():
    """The NCCL path of a point-wise split (dlopen'd libnccl, ncclCommInitRank,
    in-plan ncclAllReduce(ncclMax) on packed int64 keys): on one GPU a 1-rank
    communicator all-reduces as the identity -- the call path is real."""
    from paper_2405_05118_b200 import mdh
    nq, nr = 256, 8192
    j = spec("prl_max", [nq, nr])
    ins = prl_inputs(nq, nr, 17)
    p = mdh.rank_plan(j, 1, 0, device=0, nccl_id=mdh.nccl_unique_id(), split_dim=2)
    t = p.describe()["template"]
    assert t["nccl_allreduce"] and t["shard"]["split_kind"] == "pw", t
    (got,) = run_device(p, ins)
    ((want, _),) = mo.execute(mo.Computation.from_json(j), ins)
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [0, 1])
def test_mplan_split_from_a_multib200_configuration(dim):
    """A MultiB200 configuration's GPU-layer parts drive the split (the shard
    plans run the configuration with GPU parts 1), recombined exactly."""
    from paper_2405_05118_b200 import mdh
    from test_dev_layer_dist import multib200_config
    j = spec("matvec_fp32", [256, 512])
    comp = mo.Computation.from_json(j)
    ins = exact_inputs(comp, 8)
    mp = mdh.MultiPlan(j, 2, device_ids=[0, 0], asm="MultiB200", config=multib200_config(j["sizes"], dim, 2))
    d = mp.describe()
    assert d["split_dim"] == dim + 1 and d["split_kind"] == ("cc" if dim == 0 else "pw"), d
    (got,) = mp.run_host(ins)
    ((want, _),) = mo.execute(comp, ins)
    assert np.array_equal(got.astype(np.float64), want)
