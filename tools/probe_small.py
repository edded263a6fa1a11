"""Timing-floor probe for the small (L2-sized) routines: per-launch event time
with an L2 flush, without a flush, and back-to-back over rotating input copies.
Development aid, not the bench."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402


def ev_time(fn, reps, pre=None):
    s = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        if pre:
            pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    out.sort()
    return out[len(out) // 2]


def main():
    L2 = bench.L2_BYTES
    fw = torch.empty(3 * L2 // 4, device="cuda")
    fr = torch.zeros(3 * L2 // 4, device="cuda")

    def flush():
        fw.fill_(1.0)
        fr.sum()
    tiny = torch.zeros(1, device="cuda")
    print("empty kernel, flushed: %.2f us" % ev_time(lambda: tiny.add_(1), 20, flush))
    print("empty kernel, warm   : %.2f us" % ev_time(lambda: tiny.add_(1), 20))
    for name in sys.argv[1:] or ["matmul_resnet_fc", "matvec_fp32"]:
        plan, base, _ = bench.make_plan(name, 0)
        d_in = bench.fill(plan.empty(0), 1)
        d_out = plan.empty(1)
        inb = sum(t.numel() * t.element_size() for t in d_in)
        R = max(2, (3 * L2) // inb + 1)
        rot = [bench.fill(plan.empty(0), 2 + r) for r in range(R)]
        for _ in range(3):
            plan.run(d_in, d_out)
        f = ev_time(lambda: plan.run(d_in, d_out), 30, flush)
        w = ev_time(lambda: plan.run(d_in, d_out), 30)
        s = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 20 * R
        a.record(s)
        for i in range(steps):
            plan.run(rot[i % R], d_out)
        b.record(s)
        b.synchronize()
        r = a.elapsed_time(b) * 1e3 / steps
        d = plan.describe()
        print(json.dumps({"routine": name, "kernel": d["template"]["kernel"], "flushed_us": round(f, 2),
                          "warm_us": round(w, 2), "rotating_us": round(r, 2), "copies": R,
                          "GB/s flushed": round(d["bytes"] / f / 1e3, 1), "GB/s rotating": round(d["bytes"] / r / 1e3, 1)}))


if __name__ == "__main__":
    main()
