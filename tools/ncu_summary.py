"""Summarise ncu captures for profiles/.

    python tools/ncu_summary.py launches <launches.csv>        # per-kernel totals
    python tools/ncu_summary.py full <report.ncu-rep> [--json out.json]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list
(cold-cache, serialised: compare shares, not absolutes).  `full` prints the
DRAM/L2/occupancy/stall numbers of each kernel in a `--set full` report.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
            d["Metric Unit"], 1e-3)
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale
    total = sum(t for _, t in agg.values())
    print(f"{'launches':>8} {'total_us':>11} {'avg_us':>9} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t:11.1f} {t / c:9.1f} {t / total:6.1%}  {k}")


def full(path, json_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = f"{r[i]} {units[i]}".strip()
        out.append(rec)
        print(json.dumps(rec, indent=1))
    if json_out:
        with open(json_out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        launches(path)
    else:
        full(path, sys.argv[4] if len(sys.argv) > 4 and sys.argv[3] == "--json" else None)
