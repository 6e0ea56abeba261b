"""Statistics of D' for the bench workload (config c): how compressible the
z-delta stream is (flat 16-block chunks, zero chunks, delta histogram)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2407_21552_b200 as pdm  # noqa: E402
from paper_2407_21552_b200 import synth  # noqa: E402

cfg = bench.CFG
vol = synth.synth_volume_device(cfg["dims"], cfg["bits"], seed=cfg["seed"], nbox=cfg["nbox"])
scheme = pdm.scheme_uniform(cfg["n"], cfg["bits"])
grid = pdm.BlockGrid.for_dims(vol.dims, cfg["b"])
pset = pdm.build_pdm_set(vol, grid, scheme, cfg["mode"])
seq = bench.tf_sequence(cfg["n"], 1 << cfg["bits"], 32, cfg["seed"] + 1)
res = {}
for k, alpha in seq[::3]:
    d = pdm.update_from_tf(pset, torch.from_numpy(alpha).cuda()).device().cpu().numpy()
    d = d.reshape(-1, 16).astype(np.int16)
    delta = np.diff(d, axis=1)
    flat = (delta == 0).all(axis=1)
    hist = np.bincount((delta + 1).ravel(), minlength=3) / delta.size
    p = hist[hist > 0]
    res[k] = {"zero_frac": round(float((d == 0).mean()), 4),
              "v255_frac": round(float((d == 255).mean()), 4),
              "flat_chunks": round(float(flat.mean()), 4),
              "delta_hist": [round(float(x), 4) for x in hist],
              "entropy_bits": round(float(-(p * np.log2(p)).sum()), 3)}
print(json.dumps(res))
