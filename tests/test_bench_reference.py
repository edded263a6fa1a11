"""bench.py's reference arm (`--impl reference`): the unmodified reference's
CPU path (oracle/_ref's emitted OpenMP kernel) on the host cores, printing the
contract's JSON line -- at N=1 and under torchrun with 2 ranks (rank 0 alone
prints; the other exits 0).  CPU only."""
import json
import os
import subprocess
import sys

import pytest

from oracle import refbind

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")


def _last_json(out):
    lines = [l for l in out.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@needs_ref
def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"], cwd=REPO,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@needs_ref
def test_reference_arm_two_ranks_rank0_prints():
    env = dict(os.environ, MDHB_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29611", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3"], cwd=REPO, capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
