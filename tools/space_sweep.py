#!/usr/bin/env python3
"""Times every instance of the tuner's space (mdh_b200_tune_space) for a
BASELINE routine at full size: CUDA-event median per run (mdh_b200_time, L2
flushed), sorted.  Dev aid for choosing template defaults; writes
gpurun_out/space_<routine>.json.

    python tools/space_sweep.py jacobi3d_fp32 stencil [math]"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2405_05118_b200 import mdh  # noqa: E402


def main():
    import torch
    name, family = sys.argv[1], sys.argv[2]
    math = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    j = json.load(open(os.path.join(REPO, "specs", name + ".json")))
    sp = mdh.tune_space(j, family, math=math)
    base = mdh.Plan(j, math=math)
    d_in = base.empty(0)
    for t in d_in:
        t.uniform_(-1, 1) if t.is_floating_point() else t.random_(0, 3)
    d_out = base.empty(1)
    res = []
    t0 = time.time()
    for c in sp:
        try:
            p = mdh.Plan(j, "B200", c, math=math)
            med, ker = p.time(d_in, d_out, warmup=2, reps=5)
            t = p.describe()["template"]
            res.append({"ms": med * 1e3, "kernel_ms": ker * 1e3, "kernel": t.get("kernel"),
                        "knobs": {k: t[k] for k in ("BN", "TI", "raster_group_m", "k_split", "b_layout") if k in t},
                        "num_parts": c["num_parts"]})
            del p
        except Exception as e:  # noqa: BLE001
            res.append({"ms": float("inf"), "error": str(e)[:200], "num_parts": c["num_parts"]})
    res.sort(key=lambda r: r["ms"])
    dflt = base.time(d_in, d_out, warmup=2, reps=5)[0] * 1e3
    out = {"routine": name, "math": math, "instances": len(sp), "default_ms": dflt,
           "default_kernel": base.describe()["template"].get("kernel"), "sweep_s": time.time() - t0, "results": res}
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", f"space_{name}_{math}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name} math={math}: {len(sp)} instances, default {dflt:.4f} ms ({out['default_kernel']})")
    for r in res[:12]:
        print(f"  {r['ms']:.4f} ms  {r.get('kernel')}  {r.get('knobs')}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
