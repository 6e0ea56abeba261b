"""Box facts + oracle build time at config c (sizing the at-size parity checks)."""
import json, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import oracle
from paper_2407_21552_b200.synth import synth_boxes

out = {"nproc": os.cpu_count()}
with open("/proc/meminfo") as f:
    out["mem_total_gb"] = int(f.readline().split()[1]) / 1e6
oracle.build()
oracle.set_threads(oracle.max_threads())
out["oracle_threads"] = oracle.max_threads()
dims, bits, b, n = (1024, 1024, 1024), 16, 4, 32
boxes = synth_boxes(dims, bits, 2407, 12)
t = time.perf_counter(); vox = oracle.synth_volume(bits, dims, boxes, 2407); out["synth_s"] = time.perf_counter() - t
bounds = [(i * 2048, i * 2048 + 2047) for i in range(n)]
t = time.perf_counter(); mm = oracle.block_min_max(vox, b); out["minmax_s"] = time.perf_counter() - t
t = time.perf_counter(); occ = oracle.range_apron_presence(*mm, bounds); out["presence_s"] = time.perf_counter() - t
t = time.perf_counter(); p = oracle.distance_transform_batch(occ); out["dt_s"] = time.perf_counter() - t
print(json.dumps(out))
