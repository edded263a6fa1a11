"""Generates tests/golden/simcost.json: SimCost values of the UNMODIFIED
reference (mdh::simcost_objective, proj/src/autotuner.cpp:58-62, through
oracle/_ref) for reference-sampled configurations (ReducedSpace::sample,
tuning.cpp:354-413) of every bundled computation and for the published
fixtures, plus the reference's lowered form (lower(...).pretty(),
lowering.cpp:185-222) of the seed-1 samples.  Run here (needs /root/reference + oracle/_ref):
    python tests/golden/make_simcost_golden.py
"""
import glob
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import refbind  # noqa: E402

out = {"configs": [], "fixtures": []}
for f in sorted(glob.glob(os.path.join(HERE, "reference_data", "computations", "*.json"))):
    text = open(f).read()
    for asm in ("CUDA+WRP", "OpenMP"):
        for seed in (1, 2):
            cfg = refbind.sample_config(text, asm, seed)
            entry = {"computation": os.path.basename(f), "asm": asm, "seed": seed,
                     "config": json.loads(cfg), "simcost": refbind.simcost(text, asm, cfg)}
            if seed == 1:
                entry["lowered"] = refbind.lowered(text, asm, cfg)
            out["configs"].append(entry)
for name in ("tvm_gpu", "ppcg_gpu", "tvm_cpu", "pluto_cpu"):
    comp, cfg, asm = refbind.fixture(name)
    out["fixtures"].append({"fixture": name, "asm": asm, "simcost": refbind.simcost(comp, asm, cfg)})
json.dump(out, open(os.path.join(HERE, "simcost.json"), "w"), separators=(",", ":"))
print(len(out["configs"]), "configs,", len(out["fixtures"]), "fixtures")
