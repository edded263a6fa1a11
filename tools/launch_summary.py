"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    t = tot[r[ki][:70]]
    t[0] += 1
    t[1] += float(r[vi].replace(",", ""))
unit = rows[1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else "?"
allt = sum(v[1] for v in tot.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 1 --no-cpu  (unit {unit})")
print("(cold-cache, serialised per launch: compare shares, not absolutes)\n")
for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{k:72s} launches={n:5d} mean={t / n:12.2f} share={100 * t / allt:5.1f}%")
