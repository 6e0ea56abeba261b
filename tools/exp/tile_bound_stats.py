"""Share of (tile, selected plane) pairs a table-driven per-warp skip drops
for the bench workload (config c): per tile of T blocks and plane p, the
plane's tile minimum tmin[p] and maximum tmax[p]; for a selection S, every
block of the tile ends at most U = min_{p in S} tmax[p], so a plane q with
tmin[q] >= U cannot lower any block and is not read at all.  Also the exact
bound (tmin[q] >= max of D' over the tile) for comparison."""
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

cfg = bench.CONFIGS["c"]
vol = synth.synth_volume_device(cfg["dims"], cfg["bits"], seed=cfg["seed"], nbox=cfg["nbox"])
scheme = pdm.scheme_uniform(cfg["n"], cfg["bits"])
grid = pdm.BlockGrid.for_dims(vol.dims, cfg["b"])
pset = pdm.build_pdm_set(vol, grid, scheme, cfg["mode"])
nb = grid.num_blocks
_, timed = bench.tf_plan(cfg["n"], cfg["bits"], 32, 5, cfg["seed"] + 1)
out = {}
for tile in (256, 512, 1024, 4096):
    planes = pset.storage[:, :nb].reshape(cfg["n"], nb // tile, tile)
    tmin = planes.amin(2).int()  # [n][tiles]
    tmax = planes.amax(2).int()
    kept_tbl, kept_exact, tot = 0, 0, 0
    per_k = {}
    for picks, _ in timed:
        sel = torch.tensor([p - 1 for p in picks], device="cuda")
        U = tmax[sel].amin(0)  # [tiles]
        keep = (tmin[sel] < U[None, :])
        d = planes[sel].amin(0).amax(1).int()
        keep_x = (tmin[sel] < d[None, :])
        kept_tbl += int(keep.sum())
        kept_exact += int(keep_x.sum())
        tot += keep.numel()
        per_k[len(picks)] = round(float(keep.float().mean()), 3)
    out[tile] = {"kept_table": round(kept_tbl / tot, 3), "kept_exact": round(kept_exact / tot, 3),
                 "kept_table_by_k": per_k}
print(json.dumps(out))
