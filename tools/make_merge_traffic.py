"""profiles/merge_traffic.json from an ncu metrics CSV of
`tools/exp/merge_once.py 1 2 ... 32` (one combine_packed_flags launch per k of
the bench's 32-step TF sequence): per-k DRAM bytes (read + write) per launch.

    python tools/make_merge_traffic.py gpurun_out/r02/merge_seq.csv profiles/merge_traffic.json
"""
import csv
import io
import json
import sys


def main(src, dst):
    text = open(src).read()
    text = text[text.index('"ID"'):]  # skip ncu's preamble lines
    rows = list(csv.DictReader(io.StringIO(text)))
    per = {}
    for r in rows:
        if "combine_packed_flags" not in r["Kernel Name"]:
            continue
        per.setdefault(r["ID"], {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")),
                                                         r["Metric Unit"])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
    launches = [per[i] for i in sorted(per, key=int)]
    out = {"kernel": "combine_packed_flags_kernel<0, 0, 1> (tile skip on; k <= 4: its raw-plane path)", "per_k": {},
           "duration_us_per_k": {},
           "source": ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                      "gpu__time_duration.sum --clock-control none on tools/exp/merge_once.py "
                      "1..32 (config c, the bench's 32-step TF sequence, L2 flushed before each "
                      "merge); tools/evidence.sh")}
    for k, m in enumerate(launches, start=1):
        rd = m["dram__bytes_read.sum"][0] * scale[m["dram__bytes_read.sum"][1]]
        wr = m["dram__bytes_write.sum"][0] * scale[m["dram__bytes_write.sum"][1]]
        out["per_k"][k] = round(rd + wr)
        d = m["gpu__time_duration.sum"]
        out["duration_us_per_k"][k] = round(d[0] * scale[d[1]], 2)
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps({"launches": len(launches)}))


if __name__ == "__main__":
    main(*sys.argv[1:3])
