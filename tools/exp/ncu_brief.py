"""Brief ncu summary: duration, pipes, issue, stall breakdown (reads .ncu-rep via ncu -i)."""
import csv
import io
import subprocess
import sys

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    for row in r[2:]:
        get = lambda n: row[h.index(n)] if n in h else "?"
        print(rep.split("/")[-1], get("Kernel Name")[:50])
        for n in ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "launch__registers_per_thread", "smsp__inst_executed.sum"]:
            print("   %-70s %s" % (n, get(n)))
        items = []
        for i, name in enumerate(h):
            if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
                try:
                    items.append((float(row[i]), name[33:]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items) or 1
        print("   stalls:", ", ".join("%s %.0f%%" % (n, 100 * v / tot)
                                      for v, n in sorted(items, reverse=True)[:7]))
