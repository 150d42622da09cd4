"""Summaries of ncu output for profiles/: per-kernel metrics of a `--set full` report and the
share table of a `--metrics gpu__time_duration.sum` launch list.

  python tools/ncu_summary.py report  <file.ncu-rep>  [traffic.json]   # metrics per kernel
  python tools/ncu_summary.py launches <launches.csv>                  # per-kernel share table
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]
CLASS = {"k_colx": "col_fwd", "k_colt": "col_fwd", "k_rowd": "row", "k_dvec": "dvec", "k_colinvw": "col_inv",
         "k_transpose_n": "transpose", "k_scalars_w": "scalars"}


def _num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def report(path, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(name)
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"    {m:70s} {r[i]:>14s} {units[i]}")
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): _num(r[i]) or 0.0
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        print("    stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
        base = name.split("(")[0].split("<")[0].replace("void ", "").strip()
        cls = CLASS.get(base)
        rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = _num(r[rd]) * scale.get(units[rd], 1) + _num(r[wr]) * scale.get(units[wr], 1)
        if cls and cls not in traffic:
            traffic[cls] = b
    if traffic_out:
        with open(traffic_out, "w") as f:
            json.dump(traffic, f, indent=1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = _num(r[hdr.index("Metric Value")])
        unit = r[hdr.index("Metric Unit")]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        a = agg.setdefault(r[hdr.index("Kernel Name")], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {t:10.1f} {t / n:8.2f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        launches(sys.argv[2])
