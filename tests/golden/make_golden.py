#!/usr/bin/env python3
"""Refresh the golden fixtures under tests/golden/ from the reference tree.

Test infrastructure only.  `/root/reference` is not present on the GPU box, so
every reference-owned data file the parity tests need is committed here:

* reference_data/computations/*.json  - the 18 bundled md_hom specs
  (proj/data/computations, embedded by proj/cmake/embed_data.cmake)
* reference_data/fixtures/*.json      - the 4 published MatMul configs
  (proj/data/fixtures, parsed by parse_fixture_json, src/json_io.cpp:451-470)
* reference_data/refs/*.ref.json      - the 17 frozen known-answer vectors
  (proj/data/refs, checked by tests/test_highlevel.cpp:246-258)

These are data, not sources: no reference code is copied.  Run:

    python tests/golden/make_golden.py            # copy data files
    python tests/golden/make_golden.py --vectors  # also regenerate the
        reference-executed vectors for the BASELINE specs (needs oracle/_ref)
"""
import argparse
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_DATA = "/root/reference/proj/data"


def copy_reference_data():
    for sub in ("computations", "fixtures", "refs"):
        src = os.path.join(REF_DATA, sub)
        dst = os.path.join(HERE, "reference_data", sub)
        os.makedirs(dst, exist_ok=True)
        for name in sorted(os.listdir(src)):
            if name.endswith(".json"):
                shutil.copyfile(os.path.join(src, name), os.path.join(dst, name))
    print("copied reference data into", os.path.join(HERE, "reference_data"))


def make_vectors():
    """Run the UNMODIFIED reference (oracle/_ref) on small instances of the
    BASELINE specs (specs/*.json with sizes shrunk) and freeze input/output
    pairs in the reference's own ref-JSON format."""
    sys.path.insert(0, REPO)
    from oracle import refbind  # noqa: E402  (test infrastructure)
    from oracle import mdh_oracle as mo  # noqa: E402

    out_dir = os.path.join(HERE, "baseline_vectors")
    os.makedirs(out_dir, exist_ok=True)
    for name, sizes in SMALL_BASELINE.items():
        with open(os.path.join(REPO, "specs", name + ".json")) as f:
            spec = json.load(f)
        spec["sizes"] = sizes
        text = json.dumps(spec)
        comp = mo.Computation.from_json(text)
        inputs = mo.make_inputs(comp, seed=11)
        outs = refbind.reference_execute(text, inputs)
        doc = {"computation": spec,
               "inputs": {b.name: {"dims": list(a.shape), "data": a.ravel().tolist()}
                          for b, a in zip(comp.inputs, inputs)},
               "outputs": {b.name: {"dims": list(a.shape),
                                    "data": [None if not d else v for v, d in
                                             zip(a.ravel().tolist(), m.ravel().tolist())]}
                           for b, (a, m) in zip(comp.outputs, outs)}}
        with open(os.path.join(out_dir, name + ".vec.json"), "w") as f:
            json.dump(doc, f)
        print("wrote", name)


# BASELINE specs shrunk to oracle-friendly sizes (the divisibility structure of
# the full sizes is kept where it matters for the kernels' tiling).
SMALL_BASELINE = {
    "matvec_fp32": [64, 128],
    "jacobi3d_fp32": [8, 8, 16],
    "matmul_fp32": [32, 48, 64],
    "matmul_resnet_fc": [16, 40, 64],
    "mcc_nhwc": [2, 6, 6, 8, 3, 3, 8],
    "ccsdt_abcdef_gdab_efgc": [2, 2, 3, 2, 2, 4, 5],
    "prl_max": [16, 256],
}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--vectors", action="store_true")
    a = ap.parse_args()
    if os.path.isdir(REF_DATA):
        copy_reference_data()
    if a.vectors:
        make_vectors()
