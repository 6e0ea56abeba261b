"""Upper bound on a CTA-level plane skip for the bench workload: per tile of
8192 blocks (256 items), the share of selected planes whose tile minimum is
>= the tile maximum of D' (such a plane cannot change the tile), and the share
after folding only the plane with the smallest tile minimum first."""
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
nb = grid.num_blocks
tile = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
planes = pset.storage[:, :nb].reshape(cfg["n"], nb // tile, tile)
tmin = planes.amin(2)  # [n][tiles]
seq = bench.tf_sequence(cfg["n"], 1 << cfg["bits"], 32, cfg["seed"] + 1)
res = {}
for k, alpha in seq[::4]:
    flags = pdm.select_partitions_device(torch.from_numpy(alpha).cuda(), scheme)
    sel = torch.nonzero(flags).flatten()
    d = planes[sel].amin(0)                       # D' per tile [tiles][tile]
    dmax = d.amax(1)                               # [tiles]
    tm = tmin[sel]                                 # [k][tiles]
    ub = (tm >= dmax[None, :]).float().mean().item()
    first = planes[sel].gather(0, tm.argmin(0)[None, :, None].expand(1, -1, tile))[0]
    m1 = first.amax(1)                             # tile max after the nearest plane
    after1 = (tm >= m1[None, :]).float().mean().item()
    res[k] = {"upper_bound": round(ub, 3), "after_nearest_plane": round(after1, 3)}
print(json.dumps({"tile_blocks": tile, "skip_share": res}))
