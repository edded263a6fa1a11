#!/bin/bash
# Copy the evidence of tools/evidence.sh from gpurun_out/ into profiles/ (tag = $1)
TAG=${1:-r1}
cp gpurun_out/bench_final.json profiles/${TAG}_bench_line.json
cp gpurun_out/launches_summary.txt profiles/${TAG}_launches_summary.txt
python - "$TAG" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = [r for r in csv.reader(open("gpurun_out/launches.csv")) if len(r) > 10]
hdr = rows[0]; ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
with open(f"profiles/{tag}_launches.csv", "w") as f:
    w = csv.writer(f); w.writerow(["launch", "kernel", "gpu__time_duration.sum (ns)"])
    n = 0
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            w.writerow([n, r[ki][:90], r[vi]]); n += 1
PY
python tools/ncu_summary.py --by-routine gpurun_out ${TAG}b
for f in gpurun_out/prof_*.hot.txt; do b=$(basename $f .hot.txt); cp $f profiles/${TAG}b_${b#prof_}.hot.txt; done
