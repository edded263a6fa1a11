#!/usr/bin/env python3
"""Benchmark of the B200 MDH executor (BASELINE.json's metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--routine NAME] [--no-routines]

A step = one execution of the md_hom (one pass of the hot path) over one
batch of synthetic inputs already resident in HBM.  The headline workload is
BASELINE configs[1], Jacobi3D fp32 with a 512^3 output (specs/jacobi3d_fp32.json);
its inputs (543 MB) are larger than the 126 MB L2, so no flush is needed
between steps.  Every other §8 routine is measured too (one line, key
"routines"), each with its own roofline; those whose inputs fit in L2 are
timed with an L2 flush between runs.

Multi-GPU (torchrun, one rank per GPU): STRONG scaling of the same global
512^3 Jacobi3D -- rank r's plan is the DEV layer's shard r
(mdh_b200_rank_plan_create: 512/N output planes, its input slab carrying the
1-plane halos of the one global input, placed at distribution; a single sweep
exchanges nothing).  Every rank fills its slab from the same global
index-hashed data, so the shards' halos agree.  NCCL carries the barrier, the
max-over-ranks timing and (for point-wise splits) the in-plan all-reduce.

--impl reference times the reference's own CPU implementation of the path:
the OpenMP C kernel its code generator emits (oracle/_ref, built from
/root/reference by oracle/Makefile) on all host cores, on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = json.load(open(os.path.join(REPO, "BASELINE.json")))["metric"]
HEADLINE = "jacobi3d_fp32"
ROUTINES = ["matvec_fp32", "jacobi3d_fp32", "matmul_fp32", "matmul_fp32:tf32", "matmul_resnet_fc", "mcc_nhwc",
            "mcc_nhwc:tf32", "ccsdt_abcdef_gdab_efgc", "ccsdt_abcdef_gdab_efgc:tf32", "matmul_fp32:bf16", "mcc_nhwc:bf16",
            "ccsdt_abcdef_gdab_efgc:bf16", "prl_max", "scan_i32"]
L2_BYTES = 126 << 20


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm": j.get("hbm_gbs", 6650.0), "bf16": j.get("bf16_tflops", 1590.0),
                "bf16_sustained": j.get("bf16_tflops_sustained", 1400.0), "sm_max_mhz": j.get("sm_max_mhz", 1965.0),
                "source": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "sm_max_mhz": 1965.0, "source": "fallback"}


def spec(name):
    with open(os.path.join(REPO, "specs", name + ".json")) as f:
        return json.load(f)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Polls NVML (SM clock, throttle reasons) while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, n in self.REASONS.items():
                    if bits & b and b != 0x1:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def fill(tensors, seed):
    import torch
    g = torch.Generator(device=tensors[0].device).manual_seed(seed)
    for t in tensors:
        if t.is_floating_point():
            t.uniform_(-1, 1, generator=g)
        else:
            t.random_(0, 3, generator=g)  # PRL fields in [0,3): forces ties and matches
    return tensors


def prl_weights(d_in):
    # W (1..9) for the PRL spec: third buffer
    d_in[2].copy_(d_in[2].new_tensor([3, 5, 7, 9]))


def make_plan(name, device, world=1, rank=0, nccl_id=None):
    """Plan for routine `name` ("<spec>[:tf32]").  With world > 1 the rank's
    shard of the GLOBAL problem split over the GPU layer by the DEV layer
    (strong scaling; mdh_b200_rank_plan_create)."""
    from paper_2405_05118_b200 import mdh
    base, _, math = name.partition(":")
    m = {"": mdh.MATH_FFMA, "tf32": mdh.MATH_TF32, "bf16": mdh.MATH_BF16}[math]
    j = spec(base)
    if world > 1:
        return mdh.rank_plan(j, world, rank, device=device, nccl_id=nccl_id, math=m, int_storage=mdh.I32), \
            base, math or "ffma"
    return mdh.Plan(j, math=m, int_storage=mdh.I32, device=device), base, math or "ffma"


def fill_global(plan, seed):
    """Inputs of this rank's shard filled from ONE global array: value =
    hash(global linear index), so every rank's halo planes hold the same
    values as its neighbours' edge planes (the shard describes its slab)."""
    import torch
    d_in = plan.empty(0)
    sh = plan.describe()["template"].get("shard")
    for b, t in enumerate(d_in):
        if not t.is_floating_point():
            t.random_(0, 3)
            continue
        shape = list(t.shape)
        gshape = list(shape)
        start = 0
        if sh and sh["in"][b][0] == 0:  # the DEV layer slabs along rank 0 here
            start = sh["in"][b][1]
        inner = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        idx = torch.arange(start * inner, (start + shape[0]) * inner, device=t.device, dtype=torch.int64)
        x = (idx * 2654435761 + seed) % 4294967296
        x = ((x ^ (x >> 13)) * 1597334677) % 4294967296
        x = x ^ (x >> 16)
        t.copy_((x.to(torch.float64) / 2147483648.0 - 1.0).view(gshape).to(t.dtype))
    return d_in


def roofline_of(desc, kernel_s, pk, clock_mhz, traffic):
    """Roofline of the dominant kernel: achieved vs the peak of the resource
    that binds it.  For contractions both the compute time (FFMA or tensor
    peak) and the HBM time of the algorithmic bytes are computed and the
    larger one names the bound (CCSD(T) on the tensor cores is bound by its
    764 MB output write, not by its 27.5 GFLOP)."""
    bound = desc["bound"]
    hbm_s = desc["bytes"] / (pk["hbm"] * 1e9)

    def hbm_line(note=None):
        ach = desc["bytes"] / kernel_s / 1e9
        d = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s",
             "frac": round(ach / pk["hbm"], 4), "traffic": traffic, "peak_source": pk["source"]}
        if note:
            d["note"] = note
        return d
    if bound == "hbm":
        return hbm_line()
    if bound == "int":
        # PRL: pairs/s against the scalar integer-issue bound of the
        # ALGORITHM (3F+3 = 15 integer ops per (query, record)
        # pair at F = 4 -- compare, select, add per field, then key packing
        # and the max fold), 148 SMs x 128 lanes x clock.  frac > 1 means the
        # kernel does fewer instructions per pair than the scalar algorithm
        # (prl.cu compares 4 byte-packed fields per LOP3 / IDP.4A: 6 per pair);
        # its own issue utilisation is reported beside it, not as the roofline.
        pairs = desc["template"]["pairs"]
        F = desc["template"].get("fields", 4)
        alg_ops = 3 * F + 3
        issue = 148 * 128 * (clock_mhz or pk["sm_max_mhz"]) * 1e6
        ach = pairs / kernel_s
        peak = issue / alg_ops
        return {"bound": "int-issue", "achieved": float(f"{ach:.4g}"), "peak": float(f"{peak:.4g}"),
                "unit": "pairs/s", "frac": round(ach / peak, 4), "traffic": traffic,
                "algorithmic_ops_per_pair": alg_ops,
                "kernel_instr_per_pair": 6, "kernel_issue_frac": round(6 * ach / issue, 4)}
    if bound == "tensor":
        tf32 = desc["template"].get("math") == "tf32"
        peak = pk["bf16"] / 2.0 if tf32 else pk["bf16"]
        if hbm_s > desc["flops"] / (peak * 1e12):
            return hbm_line(f"tensor time {desc['flops'] / peak / 1e6:.1f} us < HBM time {hbm_s * 1e6:.1f} us: memory-bound")
        tflops = desc["flops"] / kernel_s / 1e12
        return {"bound": "tensor", "achieved": round(tflops, 1), "peak": round(peak, 1), "unit": "TFLOP/s",
                "frac": round(tflops / peak, 4), "traffic": traffic,
                "peak_note": "TF32 dense = 1/2 of the measured BF16 cuBLAS peak" if tf32 else "measured BF16"}
    # fp32 FFMA: 148 SMs x 128 lanes x 2 flop x clock
    peak = 148 * 128 * 2 * (clock_mhz or pk["sm_max_mhz"]) * 1e6 / 1e12
    if hbm_s > desc["flops"] / (peak * 1e12):
        return hbm_line(f"FFMA time {desc['flops'] / peak / 1e6:.1f} us < HBM time {hbm_s * 1e6:.1f} us: memory-bound")
    tflops = desc["flops"] / kernel_s / 1e12
    return {"bound": "fp32-ffma", "achieved": round(tflops, 2), "peak": round(peak, 2), "unit": "TFLOP/s",
            "frac": round(tflops / peak, 4), "traffic": traffic, "peak_note": "148 SM x 128 FMA x 2 x SM clock"}


def traffic_of(routine, kernel):
    """dram read+write bytes of this routine's dominant kernel from the
    committed ncu --set full capture (profiles/traffic.json), or None when the
    capture is of a different kernel than the one running now."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        v = json.load(open(p)).get(routine)
        if isinstance(v, dict) and kernel.split("<")[0] in v["kernel"]:
            return v["bytes"]
    return None


def time_device(plan, d_in, d_out, steps, warmup, rotate):
    """Device time of `steps` back-to-back runs of the hot path, replayed from
    one CUDA graph (so host launch overhead never enters the GPU timeline) and
    bracketed by events on the replay stream.  With `rotate` (inputs that fit
    in L2) the runs cycle over R input copies with R * bytes >= 3x L2, so every
    run reads its inputs from HBM, not from L2.  Returns (total_s, copies)."""
    import torch
    copies = [d_in]
    if rotate:
        in_bytes = sum(t.numel() * t.element_size() for t in d_in)
        R = max(2, (3 * L2_BYTES) // max(in_bytes, 1) + 1)
        for _ in range(R - 1):
            copies.append([t.clone() for t in d_in])
    for i in range(max(warmup, len(copies))):
        plan.run(copies[i % len(copies)], d_out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        for i in range(steps):
            plan.run(copies[i % len(copies)], d_out)
    for _ in range(max(1, warmup // steps)):
        g.replay()  # warm replay (graph upload, clocks)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    g.replay()
    b.record(stream)
    b.synchronize()
    tot = a.elapsed_time(b) / 1e3
    del g
    return tot, len(copies)


# ------------------------------------------------------------------ CPU baseline
def openmp_config(comp_json, threads):
    """Blocked OpenMP configuration for the reference's emitter: the outermost
    MDH layer is assigned to the COR core layer with `threads` parts along
    dim 1 (tuning.cpp:373-381 "blocked"), everything else in MM."""
    j = json.loads(comp_json)
    D = len(j["sizes"])
    n0 = j["sizes"][0]
    t = max(1, min(threads, n0))
    while n0 % t:
        t -= 1
    parts = [[t] + [1] * (D - 1), [n0 // t] + j["sizes"][1:], [1] * D, [1] * D]
    layers = ["COR", "MM", "L2", "L1"]
    ass = [[layers[l], d + 1] for l in range(4) for d in range(D)]
    return json.dumps({"num_parts": parts, "ass_de": ass, "ass_scalar": ass, "ass_re": ass}), t


def omp_threads(n):
    """omp_set_num_threads on the process's libgomp (the emitted kernels link
    the same libgomp.so.1, so this sets their team size)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        os.environ["OMP_NUM_THREADS"] = str(n)


def cpu_inputs(name, planes=None):
    """The reference's own input generator (support.hpp:32-51) on the spec,
    full size or an i-slab of `planes` planes; f64/i64 as the reference
    computes, with zeroed outputs."""
    from oracle import mdh_oracle as mo
    j = spec(name)
    if planes:
        j["sizes"][0] = planes
    text = json.dumps(j)
    comp = mo.Computation.from_json(text)
    ins = [x.astype(np.float64) if vb.type == "f64" else x for vb, x in zip(comp.inputs, mo.make_inputs(comp, 1))]
    outs = [np.zeros(s, dtype=np.float64 if vb.type == "f64" else np.int64)
            for vb, s in zip(comp.outputs, mo.output_shapes(comp))]
    return text, comp, ins, outs


def cpu_reference_kernel(name, threads, planes=None):
    """The reference's emitted OpenMP kernel (mdh::emit of a blocked OpenMP
    configuration, built with compile_and_run's flags) on the FULL workload
    (planes=None) or an i-slab.  Returns (call, description)."""
    from oracle import refbind
    text, comp, ins, outs = cpu_inputs(name, planes)
    cfg, _ = openmp_config(text, threads)
    k = refbind.EmittedKernel(text, "OpenMP", cfg)
    what = f"reference emitted OpenMP kernel (f64), {'full ' + str(comp.sizes) if not planes else str(planes) + '-plane i-slab'}"
    return (lambda: k(ins, outs)), what


def time_calls(fn, reps):
    fn()  # warm-up (first touch of the outputs, thread team start)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def cpu_baseline_line(name, reps=3):
    """cpu_baseline of our arm: the reference's emitted OpenMP kernel on the
    same full workload with every host thread (the value), beside it the same
    kernel on one thread and the single-threaded reference_execute
    (highlevel.cpp:110-113) on an 8-plane slab, extrapolated and labelled so."""
    from oracle import refbind
    full_bytes = bytes_of_spec(name)
    threads = os.cpu_count() or 1
    try:
        call, what = cpu_reference_kernel(name, threads)
        omp_threads(threads)
        s_all = time_calls(call, reps)
        omp_threads(1)
        s_one = time_calls(call, 1)
        omp_threads(threads)
        del call
        _, comp, ins, _ = cpu_inputs(name, 8)
        text = json.dumps(comp.to_json())
        t0 = time.perf_counter()
        refbind.reference_execute(text, ins)
        s_ref = (time.perf_counter() - t0) * spec(name)["sizes"][0] / 8
        return {"value": round(full_bytes / s_all / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                "sample": f"{what}, {threads} threads, median of {reps}; GB/s counted with the fp32 algorithmic "
                          "bytes of the same points (same config as the GPU arm)",
                "ms_per_step": round(s_all * 1e3, 2), "host_cpu": host_cpu(),
                "one_thread": {"value": round(full_bytes / s_one / 1e9, 3), "ms_per_step": round(s_one * 1e3, 2),
                               "sample": what + ", 1 thread"},
                "reference_execute": {"value": round(full_bytes / s_ref / 1e9, 4), "s_per_step": round(s_ref, 2),
                                      "sample": "mdh::reference_execute (single-threaded by contract), 8-plane "
                                                "i-slab, extrapolated to the full workload"}}
    except Exception as e:  # reference not built: the C restatement, 1 thread, on a slab
        from oracle import mdh_oracle as mo
        _, comp, ins, _ = cpu_inputs(name, 8)
        t0 = time.perf_counter()
        mo.execute(comp, ins, mo.pw_outer_plan(comp))
        s = (time.perf_counter() - t0) * spec(name)["sizes"][0] / 8
        return {"value": round(full_bytes / s / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "port",
                "sample": f"oracle C restatement (f64, 1 thread) on an 8-plane slab, extrapolated "
                          f"(reference unavailable: {e})"}


def host_cpu():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--routine", default=HEADLINE)
    ap.add_argument("--no-routines", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        # the reference's own CPU implementation of the path, on the SAME
        # workload as our arm (full size), every host thread, one run per step
        if rank != 0:
            return
        base = args.routine.partition(":")[0]
        threads = os.cpu_count() or 1
        omp_threads(threads)
        call, what = cpu_reference_kernel(base, threads)
        for _ in range(max(1, args.warmup)):
            call()
        runs = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            call()
            runs.append(time.perf_counter() - t0)
        tot = sum(runs)
        per = tot / len(runs)
        value = bytes_of_spec(base) / per / 1e9
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(per * 1e3, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator)",
                "impl": "reference",
                "config": {"workload": f"{base} {spec(base)['sizes']} (full, same as the GPU arm)", "threads": threads,
                           "host_cpu": host_cpu()},
                "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                                 "sample": what + f", {threads} threads; GB/s counted with the fp32 algorithmic "
                                                  "bytes of the same points"},
                "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if world > 1:
        import torch.distributed as dist
        # MDHB_BENCH_BACKEND=gloo + fewer GPUs than ranks exercises the N>1
        # path on one GPU (test aid); the real run is NCCL, one rank per GPU
        backend = os.environ.get("MDHB_BENCH_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend)
    device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    pk = peaks()

    # ---- headline: device-resident steps
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        from paper_2405_05118_b200 import mdh
        box = [mdh.nccl_unique_id() if rank == 0 and dist.get_backend() == "nccl" else None]
        dist.broadcast_object_list(box, src=0)
        nccl_id = box[0]
    plan, base, math = make_plan(args.routine, device, world, rank, nccl_id)
    desc = plan.describe()
    d_in = fill_global(plan, 1234)
    if base == "prl_max":
        prl_weights(d_in)
    d_out = plan.empty(1)
    in_bytes = sum(t.numel() * t.element_size() for t in d_in)
    rotate = in_bytes < 2 * L2_BYTES
    sync_all(world)
    with ClockSampler(device) as clk:
        tot, copies = time_device(plan, d_in, d_out, args.steps, args.warmup, rotate)
    tot = max_over_ranks(tot, world)
    ms = tot / args.steps * 1e3
    gdesc = desc if world == 1 else make_plan(args.routine, device)[0].describe()  # the global problem's work
    value = gdesc["bytes"] / (tot / args.steps) / 1e9 if desc["bound"] == "hbm" else \
        gdesc["flops"] / (tot / args.steps) / 1e9
    unit = "GB/s" if desc["bound"] == "hbm" else "GFLOP/s"
    kernel_s = tot / args.steps
    clocks = clk.summary()
    roof = roofline_of(desc, kernel_s, pk, clocks["sm_mhz"], traffic_of(args.routine, desc["template"]["kernel"]))

    # ---- e2e through the C ABI with pinned host buffers
    e2e = e2e_measure(plan, d_in, max(3, min(args.steps, 10)), world, gdesc)

    line = {"metric": METRIC, "value": round(value, 2), "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if base != "prl_max" else "i32",
            "data": "synthetic (one global array, uniform(-1,1) fp32 from a hash of the global index)",
            "config": {"workload": f"{base} {spec(base)['sizes']} ({math}), global problem over all GPUs",
                       "family": desc["family"],
                       "kernel": desc["template"]["kernel"],
                       "parallelism": (f"DEV layer: ++ dim {desc['template']['shard']['split_dim']} split into "
                                       f"{world} shards (strong), rank plans" if world > 1 else "single GPU"),
                       "l2": f"inputs rotated over {copies} copies (> 3x L2)" if rotate else
                       f"inputs ({in_bytes >> 20} MB) larger than L2",
                       "timing": "K runs replayed from one CUDA graph, CUDA events on the replay stream"},
            "roofline": roof, "clocks": clocks, "e2e": e2e,
            "gpu_launches": plan.launches * args.steps}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_line(base)
    if not args.no_routines and world == 1:
        line["routines"] = routines_table(device, pk, world, exclude=args.routine)
        line["gpu_launches"] += sum(r.get("launches", 0) for r in line["routines"])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def bytes_of_spec(name):
    from oracle import mdh_oracle as mo  # shapes only (the CPU sample accounting)
    comp = mo.Computation.from_json(spec(name))
    n = sum(int(np.prod(s)) for s in mo.input_shapes(comp)) + sum(int(np.prod(s)) for s in mo.output_shapes(comp))
    return 4 * n


def sync_all(world):
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def e2e_measure(plan, d_in, reps, world, gdesc=None):
    """Host (pinned) inputs -> mdh_b200_run_host -> host outputs, wall clock."""
    import torch
    h_in = [t.cpu().pin_memory() for t in d_in]
    tdt = {0: torch.float32, 1: torch.float64, 2: torch.int32, 3: torch.int64}
    h_out = [torch.empty(o["shape"], dtype=tdt[o["dtype"]]).pin_memory() for o in plan.outputs]
    np_in = [t.numpy() for t in h_in]
    np_out = [t.numpy() for t in h_out]
    plan.run_host(np_in, np_out)  # warm-up (allocates the plan's device buffers)
    sync_all(world)
    t0 = time.perf_counter()
    for _ in range(reps):
        plan.run_host(np_in, np_out)
    dt = (time.perf_counter() - t0) / reps
    dt = max_over_ranks(dt, world)
    desc = gdesc or plan.describe()
    work = desc["bytes"] if desc["bound"] == "hbm" else desc["flops"]
    unit = "GB/s" if desc["bound"] == "hbm" else "GFLOP/s"
    return {"value": round(work / dt / 1e9, 2), "unit": unit,
            "h2d_bytes_per_step": int(sum(a.nbytes for a in np_in)),
            "d2h_bytes_per_step": int(sum(a.nbytes for a in np_out)), "ms_per_step": round(dt * 1e3, 3)}


def routines_table(device, pk, world, exclude):
    import torch
    out = []
    for name in ROUTINES:
        if name == exclude:
            continue
        try:
            plan, base, math = make_plan(name, device)
        except Exception as e:
            out.append({"routine": name, "error": str(e)})
            continue
        desc = plan.describe()
        d_in = fill(plan.empty(0), 99)
        if base == "prl_max":
            prl_weights(d_in)
        d_out = plan.empty(1)
        in_bytes = sum(t.numel() * t.element_size() for t in d_in)
        heavy = desc["flops"] > 1e11 or base == "prl_max"
        steps = 3 if heavy else 50
        tot, copies = time_device(plan, d_in, d_out, steps, 3, in_bytes < 2 * L2_BYTES)
        k = tot / steps
        roof = roofline_of(desc, k, pk, None, traffic_of(name, desc["template"]["kernel"]))
        ent = {"routine": name, "family": desc["family"], "kernel": desc["template"]["kernel"],
               "ms": round(k * 1e3, 4), "GB/s": round(desc["bytes"] / k / 1e9, 1),
               "GFLOP/s": round(desc["flops"] / k / 1e9, 1), "roofline": roof, "launches": plan.launches * steps,
               "input_copies": copies}
        if base == "prl_max":
            ent["pairs_per_s"] = desc["template"]["pairs"] / k
        out.append(ent)
        del plan, d_in, d_out
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
