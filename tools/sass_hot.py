"""Top SASS instructions of an ncu report's source page by executed count and
by stall samples (development aid): python tools/sass_hot.py rep.ncu-rep [N] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
args = ["ncu", "-i", rep, "--page", "source", "--csv"]
if len(sys.argv) > 3:
    args += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# a report may hold several kernels: each starts with a "Kernel Name" row
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
b = blocks[-1]
hdr = b["rows"][0]
ie, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
data = [r for r in b["rows"][1:] if len(r) > ie]
tot = sum(float(r[ie] or 0) for r in data)
tots = sum(float(r[ss] or 0) for r in data)
print(b["name"], "instructions", tot, "stall samples", tots)
print("-- by stall samples")
for r in sorted(data, key=lambda r: -float(r[ss] or 0))[:n]:
    print(f"{r[0]:>6} {float(r[ss] or 0):7.0f} {float(r[ie] or 0):9.0f}  {r[src][:90]}")
