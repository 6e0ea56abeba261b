"""Host decode throughput on the GPU box's CPU: sparse (zero / mixed / coded
regions) vs delta vs nibble expansion of a 16.8 MB map."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))
from paper_2407_21552_b200 import _lib  # noqa: E402
from test_host_api import _sparse_regions  # noqa: E402

L = _lib.load_library()
nb = 1 << 24
chunks = nb // 16
rng = np.random.default_rng(0)
import torch  # noqa: E402

out = torch.empty(nb, dtype=torch.uint8, pin_memory=True).numpy()


def t(fn, reps=30):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(float(np.median(ts)) * 1e3, 4)


res = {}
for name, p in (("zero", [1, 0, 0]), ("mixed", [0.2, 0.4, 0.4]), ("coded", [0, 0, 1])):
    kind = rng.choice(3, 64 * 256, p=p)
    steps = rng.integers(-1, 2, (64 * 256, 16))
    steps[kind != 2] = 0
    start = rng.choice([1, 37, 254], 64 * 256)
    start[kind == 0] = 0
    vals = np.clip(start[:, None] + np.cumsum(steps, 1) - steps[:, :1], 0, 255)
    regions = np.ascontiguousarray(np.tile(_sparse_regions(vals), (chunks // 64 // 256, 1)))
    res["sparse_" + name] = t(lambda: L.pdm_unpack_sparse_host(regions.ctypes.data, nb,
                                                               out.ctypes.data))
    if name == "coded":
        v = np.tile(vals, (chunks // (64 * 256), 1))
        d = np.diff(v, axis=1) + 1
        codes = (d << (2 * np.arange(15))).sum(1).astype(np.uint32)
        base = v[:, 0].astype(np.uint8)
        res["delta"] = t(lambda: L.pdm_unpack_delta_host(codes.ctypes.data, base.ctypes.data,
                                                          nb, out.ctypes.data))
res["memset"] = t(lambda: out.fill(0))
print(json.dumps(res))
