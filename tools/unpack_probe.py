"""Host expansion cost of a packed D' (pdm_unpack_packed_host) at config c."""
import sys, time, json
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_21552_b200 import _lib
L = _lib.load_library()
nb = 256 ** 3
chunks = 2 * (-(-nb // 32))
rng = np.random.default_rng(0)
nib = rng.integers(0, 256, chunks * 8, dtype=np.uint8)
base = rng.integers(0, 200, chunks, dtype=np.uint8)
out = np.empty(nb, np.uint8)
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    L.pdm_unpack_packed_host(nib.ctypes.data, base.ctypes.data, nb, out.ctypes.data)
    ts.append((time.perf_counter() - t0) * 1e3)
import os
print(json.dumps({"unpack_ms_median": round(float(np.median(ts)), 4), "min": round(min(ts), 4),
                  "cpus": os.cpu_count()}))
