"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"]


def summary(path):
    """Summary of the longest launch in the report (the routine's dominant kernel)."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ti = hdr.index("gpu__time_duration.sum")

    def dur(r):
        try:
            return float(r[ti].replace(",", ""))
        except ValueError:
            return -1.0
    vals = max(rows[2:], key=dur)
    d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
         "launches_in_report": len(rows) - 2}
    for k in KEYS:
        if k in hdr:
            d[k] = vals[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
    stalls = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v or 0))
              for h, v in zip(hdr, vals) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
    d["top_stalls"] = sorted(stalls, key=lambda x: -x[1])[:6]
    others = [h for h in hdr if "tensor" in h or "tcgen05" in h or "utc" in h.lower()]
    d["tensor_metrics"] = {h: vals[hdr.index(h)] for h in others[:12]}
    return d


def dram_bytes(d):
    """dram read + write of the summarised launch, in bytes."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = d[k].split()
        tot += float(v.replace(",", "")) * scale[u]
    return int(tot)


if __name__ == "__main__":
    # tools/ncu_summary.py report.ncu-rep ...            -> print
    # tools/ncu_summary.py --by-routine DIR TAG          -> DIR/prof_<routine>.ncu-rep into
    #                                                       profiles/<TAG>_ncu_<routine>.json + traffic.json
    if sys.argv[1] == "--by-routine":
        import glob
        import os
        src, tag = sys.argv[2], sys.argv[3]
        repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        tp = os.path.join(repo, "profiles", "traffic.json")
        traffic = json.load(open(tp)) if os.path.exists(tp) else {}
        traffic = {k: v for k, v in traffic.items() if isinstance(v, dict)}
        for rep in sorted(glob.glob(os.path.join(src, "prof_*.json"))):
            routine = os.path.basename(rep)[5:-5].replace("__", ":")
            d = json.load(open(rep))
            d["routine"] = routine
            with open(os.path.join(repo, "profiles", f"{tag}_ncu_{routine.replace(':', '_')}.json"), "w") as f:
                json.dump(d, f, indent=1)
            traffic[routine] = {"kernel": d["kernel"], "bytes": dram_bytes(d)}
            print(routine, d["kernel"], d["gpu__time_duration.sum"], traffic[routine]["bytes"])
        with open(tp, "w") as f:
            json.dump(traffic, f, indent=1)
    else:
        for p in sys.argv[1:]:
            print(json.dumps(summary(p), indent=1))
