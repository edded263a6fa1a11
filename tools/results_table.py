#!/usr/bin/env python3
"""BASELINE.md section 3's results table from a bench line (bench.py JSON) and
the CPU table (tools/cpu_table.py JSON).  Usage:
    python tools/results_table.py profiles/r2i_bench_line.json profiles/r2_cpu_table.json"""
import json
import sys

PARITY = {
    "matvec_fp32": "exact (full size, k/4) + 1e-5 sqrt(K)",
    "jacobi3d_fp32": "U(-1,1) tol, full-size planes + linearity",
    "matmul_fp32": "exact rows at 8192^3 + U(-1,1) bounds (FFMA/TF32/BF16)",
    "matmul_resnet_fc": "exact, full size",
    "mcc_nhwc": "exact images 0/255 + U(-1,1) bounds (FFMA/TF32/BF16)",
    "ccsdt_abcdef_gdab_efgc": "exact slices + U(-1,1) bounds (FFMA/TF32/BF16)",
    "prl_max": "bit-exact (sampled full-size queries, brute force)",
}
LABEL = {
    "matvec_fp32": "MatVec FP32 4096^2", "jacobi3d_fp32": "Jacobi3D FP32 512^3", "matmul_fp32": "MatMul 8192^3",
    "matmul_resnet_fc": "MatMul FC 16x1000x2048", "mcc_nhwc": "MCC conv2_x N=256",
    "ccsdt_abcdef_gdab_efgc": "CCSD(T) 24^6 x 72", "prl_max": "PRL 2^15 x 2^20",
}


def main():
    bench = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    cpu = json.load(open(sys.argv[2]))
    rows = {bench["config"]["workload"].split()[0]: [{"routine": bench["config"]["workload"].split()[0],
                                                      "kernel": bench["config"]["kernel"],
                                                      "ms": bench["ms_per_step"], "roofline": bench["roofline"]}]}
    for r in bench.get("routines", []):
        rows.setdefault(r["routine"].split(":")[0], []).append(r)
    th = cpu["threads"]
    print(f"| Config | B200 kernel(s), 1 GPU | measured | % roofline | CPU `reference_execute` 1 thread (s) | "
          f"CPU emitted OpenMP, {th} / 1 threads (s) | Parity |")
    print("|---|---|---|---|---|---|---|")
    for name, label in LABEL.items():
        meas, frac, kern = [], [], []
        for r in rows.get(name, []):
            math = r["routine"].split(":")[1] if ":" in r["routine"] else ("int" if name == "prl_max" else "fp32")
            rf = r["roofline"]
            unit = rf.get("unit", "")
            ach = rf.get("achieved")
            meas.append(f"{math}: {r['ms']:.4g} ms = {ach:.4g} {unit}")
            frac.append(f"{math}: {rf.get('frac', 0):.3f} ({rf.get('bound')})")
            kern.append(f"`{r['kernel']}`")
        c = cpu["rows"].get(name, {})
        ext = " (extrap.)" if c.get("extrapolated") else ""
        full = json.load(open(f"specs/{name}.json"))["sizes"]
        rext = " (extrap.)" if c and c["reference_execute_sizes"] != full else ""
        cref = f"{c['reference_execute_s']:.3g}{rext}" if c else "—"
        comp = f"{c['omp_all_s']:.3g} / {c['omp_one_s']:.3g}{ext}" if c else "—"
        print(f"| {label} | {'<br>'.join(kern)} | {'<br>'.join(meas)} | {'<br>'.join(frac)} | {cref} | {comp} | "
              f"{PARITY.get(name, '')} |")


if __name__ == "__main__":
    main()
