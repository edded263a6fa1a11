"""bench.py contract on one GPU: the single-GPU JSON line, and the N>1
(torchrun) strong-scaling path (DEV-layer rank plans on one global problem)
exercised with 2 ranks sharing the GPU over gloo."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    out = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--no-routines", "--no-cpu"],
                         cwd=REPO, capture_output=True, text=True, timeout=600).stdout
    d = _last_json(out)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["value"] > 0 and d["gpu_launches"] >= 5
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_strong_scaling_path():
    env = dict(os.environ, MDHB_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3",
           "--no-routines"]
    p = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    d = _last_json(p.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and "2 shards" in d["config"]["parallelism"]
    # whole-job value over the GLOBAL problem: the same algorithmic bytes as one GPU
    assert d["config"]["workload"].startswith("jacobi3d_fp32 [512, 512, 512]")
