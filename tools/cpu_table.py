#!/usr/bin/env python3
"""CPU side of BASELINE.md's results table, measured on the host it runs on
(the GPU box's host when run under gpurun): per BASELINE routine

  * mdh::reference_execute (highlevel.cpp:110-113; single-threaded by
    contract) on a reduced-size instance of the same spec, extrapolated to the
    full size by the point count;
  * the reference's emitted OpenMP kernel (mdh::emit of a blocked OpenMP
    configuration, compile_and_run's flags) on every host thread and on one
    thread, at full size where a run takes under a few seconds, else on an
    i-slab extrapolated by the point count.

Both are the unmodified reference (oracle/_ref), f64/i64 as it computes.
Writes gpurun_out/cpu_table.json and prints a markdown table."""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from oracle import mdh_oracle as mo  # noqa: E402
from oracle import refbind  # noqa: E402

# routine -> (sizes for reference_execute, sizes for the emitted kernel)
CASES = {
    "matvec_fp32": ([4096, 4096], [4096, 4096]),
    "jacobi3d_fp32": ([8, 512, 512], [512, 512, 512]),
    "matmul_fp32": ([1, 8192, 8192], [32, 8192, 8192]),
    "matmul_resnet_fc": ([16, 1000, 2048], [16, 1000, 2048]),
    "mcc_nhwc": ([1, 56, 56, 64, 3, 3, 64], [32, 56, 56, 64, 3, 3, 64]),
    "ccsdt_abcdef_gdab_efgc": ([1, 4, 24, 24, 24, 24, 72], [8, 24, 24, 24, 24, 24, 72]),
    "prl_max": ([16, 1048576], [256, 1048576]),
}


def points(sizes):
    return float(np.prod(np.array(sizes, dtype=np.float64)))


def inputs(name, sizes):
    j = bench.spec(name)
    j["sizes"] = list(sizes)
    text = json.dumps(j)
    comp = mo.Computation.from_json(text)
    ins = [x.astype(np.float64) if vb.type == "f64" else x for vb, x in zip(comp.inputs, mo.make_inputs(comp, 1))]
    outs = [np.zeros(s, dtype=np.float64 if vb.type == "f64" else np.int64)
            for vb, s in zip(comp.outputs, mo.output_shapes(comp))]
    return text, ins, outs


def main():
    threads = os.cpu_count() or 1
    rows = {}
    for name, (ref_sizes, omp_sizes) in CASES.items():
        full = bench.spec(name)["sizes"]
        text, ins, _ = inputs(name, ref_sizes)
        t0 = time.perf_counter()
        refbind.reference_execute(text, ins)
        s_ref = (time.perf_counter() - t0) * points(full) / points(ref_sizes)
        del ins
        text, ins, outs = inputs(name, omp_sizes)
        cfg, t = bench.openmp_config(text, threads)
        k = refbind.EmittedKernel(text, "OpenMP", cfg)
        scale = points(full) / points(omp_sizes)
        bench.omp_threads(threads)
        s_all = bench.time_calls(lambda: k(ins, outs), 3) * scale
        bench.omp_threads(1)
        s_one = bench.time_calls(lambda: k(ins, outs), 1) * scale
        bench.omp_threads(threads)
        rows[name] = {"reference_execute_s": s_ref, "reference_execute_sizes": ref_sizes,
                      "omp_all_s": s_all, "omp_one_s": s_one, "omp_sizes": omp_sizes, "omp_parts": t,
                      "threads": threads, "extrapolated": scale != 1.0}
        print(name, json.dumps(rows[name]), flush=True)
        del ins, outs, k
    out = {"host_cpu": bench.host_cpu(), "threads": threads, "rows": rows}
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "cpu_table.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"| routine | reference_execute 1 thread (s) | emitted OpenMP {threads} threads (s) | emitted OpenMP 1 thread (s) |")
    for n, r in rows.items():
        ext = " (extrapolated)" if r["extrapolated"] else ""
        print(f"| {n} | {r['reference_execute_s']:.3g} | {r['omp_all_s']:.3g}{ext} | {r['omp_one_s']:.3g}{ext} |")


if __name__ == "__main__":
    main()
