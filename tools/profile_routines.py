"""Runs every bench routine's hot path exactly once (after one untimed warm-up
on the same inputs) so that one `ncu --set full` pass captures each product
kernel once.  Development aid: numbers printed under ncu are never bench values.

    ncu --set full --clock-control none --import-source on \
        -k regex:'star7|gemv|sgemm|skinny|tc_gemm|prl_|vm_|scan' -o gpurun_out/all \
        python tools/profile_routines.py [routine ...]

`tools/ncu_summary.py --by-routine gpurun_out/all.ncu-rep` then writes
profiles/ncu_<routine>.json and profiles/traffic.json.
"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402


def main():
    names = sys.argv[1:] or bench.ROUTINES
    for name in names:
        plan, base, _ = bench.make_plan(name, 0)
        d_in = bench.fill(plan.empty(0), 99)
        if base == "prl_max":
            bench.prl_weights(d_in)
        d_out = plan.empty(1)
        # the warm-up launch is excluded by ncu's -k filter only if it names the
        # same kernel, so mark the boundary with a torch kernel and skip nothing:
        # the summary keeps the LAST capture of each kernel per routine
        plan.run(d_in, d_out)
        torch.cuda.synchronize()
        plan.run(d_in, d_out)
        torch.cuda.synchronize()
        print(name, plan.describe()["template"]["kernel"], flush=True)
        del plan, d_in, d_out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
