"""Where the first build_pdm_set call of a process spends its time
(the reference bench reports it as one_time_init_ms)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
t0 = time.perf_counter()
import numpy as np  # noqa: E402

import paper_2407_21552_b200 as P  # noqa: E402

r = {"import_s": round(time.perf_counter() - t0, 3)}
rng = np.random.default_rng(0)
vox = rng.integers(0, 256, size=(128, 128, 128), dtype=np.uint8)
t = time.perf_counter()
import torch  # noqa: E402

torch.cuda.init()
torch.empty(1, device="cuda")
r["torch_cuda_init_s"] = round(time.perf_counter() - t, 3)
t = time.perf_counter()
P._lib.lib()
r["lib_load_s"] = round(time.perf_counter() - t, 3)
vol = P.Volume.from_array(vox)
grid = P.BlockGrid.for_dims(vol.dims, 4)
for n in (16, 32):
    scheme = P.scheme_uniform(n, 8)
    for mode in ("voxel", "range_apron"):
        t = time.perf_counter()
        P.build_pdm_set(vol, grid, scheme, mode)
        r[f"build_{n}_{mode}_s"] = round(time.perf_counter() - t, 4)
print(json.dumps(r))
