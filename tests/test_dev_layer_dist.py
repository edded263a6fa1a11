"""The C++ DEV layer's split rule on CPU (host only): world_size-2 gloo
process groups take their shard from mdh_b200_shard_spec (the same code path
mdh_b200_rank_plan_create uses), run the oracle on it over their slabs of
the global inputs, and recombine -- point-wise shards by an all-reduce with
the dimension's operator, ++ shards by gathering the output slabs.  The
result must equal the unsplit oracle exactly.  (The CUDA kernels on each
shard: tests/test_gpu_dev_layer.py.)"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import spec
from oracle import mdh_oracle as mo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(name, comp):
    if name == "prl_max":
        rng = np.random.default_rng(3)
        return [rng.integers(0, 3, s).astype(np.int64) for s in mo.input_shapes(comp)[:2]] + [np.array([3, 5, 7, 9])]
    return mo.make_inputs(comp, 3)


OPS = {"+": "SUM", "max": "MAX", "min": "MIN", "*": "PRODUCT"}


def _worker(rank, world, port, spec_json, split_dim, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2405_05118_b200 import mdh
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        j = json.loads(spec_json)
        full = mo.Computation.from_json(j)
        ins = _inputs(j["name"], full)
        sh = mdh.shard_spec(j, world, rank, split_dim=split_dim)
        comp = mo.Computation.from_json(sh["computation"])
        shapes = mo.input_shapes(comp)
        mine = []
        for x, (r, st), shp in zip(ins, sh["shard"]["in"], shapes):
            if r < 0:
                mine.append(x)
            else:
                idx = [slice(None)] * x.ndim
                idx[r] = slice(st, st + shp[r])
                mine.append(np.ascontiguousarray(x[tuple(idx)]))
        outs = mo.execute(comp, mine)
        res = []
        for (vals, _), (r, st) in zip(outs, sh["shard"]["out"]):
            t = torch.from_numpy(np.ascontiguousarray(vals))
            if sh["shard"]["split_kind"] == "pw":
                op = j["combine"][sh["shard"]["split_dim"] - 1].split(":")[1]
                dist.all_reduce(t, op=getattr(dist.ReduceOp, OPS[op]))
                res.append(t.numpy())
            else:
                parts = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                res.append(torch.cat(parts, dim=r).numpy())
        if rank == 0:
            want = mo.execute(full, ins)
            q.put([bool(np.array_equal(g, w[0])) for g, w in zip(res, want)])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,sizes,split_dim", [
    ("prl_max", [32, 512], 2),              # record split: max of packed keys
    ("prl_max", [32, 512], 1),              # query split
    ("matvec_fp32", [16, 64], 2),           # k split: sum
    ("matvec_fp32", [16, 64], 0),           # automatic: rows
    ("jacobi3d_fp32", [8, 6, 5], 0),        # z slabs with ghost planes
    ("mcc_nhwc", [4, 4, 4, 8, 3, 3, 4], 1), # images
    ("ccsdt_abcdef_gdab_efgc", [2, 2, 2, 2, 2, 2, 4], 0),
])
def test_world2_cpp_split_recombines_exactly(name, sizes, split_dim):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    j = json.dumps(spec(name, sizes))
    procs = [ctx.Process(target=_worker, args=(r, 2, port, j, split_dim, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(60)
    assert all(ok) and all(p.exitcode == 0 for p in procs), ok


def multib200_config(sizes, dim, parts):
    """A MultiB200 configuration (ASM layers HM, DM, SM, RM, GPU, SMX, WRP, CC;
    MDH layer l on ASM layer l): everything on HM except `parts` GPU-layer
    parts of dimension `dim` (0-based)."""
    L = 8
    rows = [[1] * len(sizes) for _ in range(L)]
    rows[0] = list(sizes)
    rows[0][dim] //= parts
    rows[4][dim] = parts
    return json.dumps({"num_parts": rows})


@pytest.mark.parametrize("dim", [0, 1])
def test_split_from_a_multib200_configuration(dim):
    """The GPU-layer parts of a MultiB200 configuration choose the split
    (the reference's MultiGPU ASM, asm_model.cpp:36-37), and the shard's
    configuration keeps every other part with GPU parts 1."""
    from paper_2405_05118_b200 import mdh
    j = spec("matvec_fp32", [64, 128])
    cfg = multib200_config(j["sizes"], dim, 4)
    assert mdh.validate_config(j, "MultiB200", cfg) == ""
    for r in range(4):
        sh = mdh.shard_spec(j, 4, r, config=cfg)
        assert sh["shard"]["split_dim"] == dim + 1
        assert sh["computation"]["sizes"][dim] == j["sizes"][dim] // 4
        gpu_row = sh["config"]["num_parts"][4]
        assert all(x == 1 for x in gpu_row)
