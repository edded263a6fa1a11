"""The N>1 path on CPU: world_size-2 gloo process groups run shards of an
md_hom (computed by the oracle -- this exercises the host-side split and the
collectives, not the kernels) and recombine them: ++ shards by gathering the
output slabs, point-wise shards by an all-reduce with the dim's operator.
The recombined result must equal the unsplit oracle result exactly."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import bundled, spec
from oracle import mdh_oracle as mo
from paper_2405_05118_b200.shard import combine_op, shard_spec, take


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec_json, dim, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = mo.Computation.from_json(spec_json)
        ins = mo.make_inputs(full, seed)
        sub, in_sl, out_sl, op = shard_spec(spec_json, dim, world, rank)
        comp = mo.Computation.from_json(sub)
        shapes = mo.input_shapes(comp)
        my_ins = [np.ascontiguousarray(take(x, sl, shp[sl[0]] if sl else None)) for x, sl, shp in
                  zip(ins, in_sl, shapes)]
        outs = mo.execute(comp, my_ins)
        results = []
        for (vals, dfd), sl in zip(outs, out_sl):
            t = torch.from_numpy(np.ascontiguousarray(vals))
            if op is not None:  # point-wise shard: fold with the dim's operator
                dist.all_reduce(t, op=combine_op(dist, op))
                results.append(t.numpy())
            else:               # ++ shard: gather the slabs in rank order
                parts = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                results.append(torch.cat(parts, dim=sl[0] if sl else 0).numpy())
        if rank == 0:
            q.put([r.tolist() for r in results])
    finally:
        dist.destroy_process_group()


def _run(spec_json, dim, seed=3, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec_json, dim, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = mo.Computation.from_json(spec_json)
    want = mo.execute(full, mo.make_inputs(full, seed))
    return got, want


@pytest.mark.parametrize("name,sizes,dim", [
    ("jacobi3d_fp32", [8, 6, 6], 0),       # z-slab split with halo planes
    ("matvec_fp32", [16, 32], 0),          # row split, v replicated
    ("mcc_nhwc", [4, 4, 4, 4, 3, 3, 4], 0),  # image split, filter replicated
])
def test_concat_split_two_ranks(name, sizes, dim):
    got, want = _run(json.dumps(spec(name, sizes)), dim)
    for g, (w, d) in zip(got, want):
        assert np.array_equal(np.array(g), w)


@pytest.mark.parametrize("name,sizes,dim", [
    ("prl_max", [8, 64], 1),               # record split: max over packed int64 keys
    ("matvec_fp32", [8, 32], 1),           # k split: sum of partial dot products
])
def test_pointwise_split_two_ranks(name, sizes, dim):
    got, want = _run(json.dumps(spec(name, sizes)), dim)
    for g, (w, d) in zip(got, want):
        assert np.array_equal(np.array(g), w)


def test_histogram_idx_stays_global():
    """idx() of the split dim is rebased so index-dependent scalars agree."""
    j = bundled("genhisto", [8, 6])
    got, want = _run(json.dumps(j), 1)
    for g, (w, d) in zip(got, want):
        assert np.array_equal(np.array(g), w)


def test_non_divisible_split_rejected():
    with pytest.raises(ValueError):
        shard_spec(spec("matvec_fp32", [10, 8]), 0, 4, 0)
