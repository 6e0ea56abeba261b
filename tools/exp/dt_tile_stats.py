"""How much of the DT's sweep work is on constant tiles (config c): after
pass x, the share of y-pass warp tiles (32 z x all y of one (p, x)) whose
values are all 255 or all 0, and in the final maps the share of z-pass warp
tiles (32 rows) that are constant (their input rows then were too)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2407_21552_b200 as pdm  # noqa: E402
from paper_2407_21552_b200 import _lib, synth  # noqa: E402

cfg = bench.CONFIGS["c"]
vol = synth.synth_volume_device(cfg["dims"], cfg["bits"], seed=cfg["seed"], nbox=cfg["nbox"])
scheme = pdm.scheme_uniform(cfg["n"], cfg["bits"])
grid = pdm.BlockGrid.for_dims(vol.dims, cfg["b"])
mask = pdm.acceleration.partition_mask(vol, grid, scheme, cfg["mode"])
n = scheme.n
bx, by, bz = grid.bdims
pitch = pdm.device.plane_pitch(grid.num_blocks)
st = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
L = _lib.lib()
_lib.check(L.pdm_dt_pass_x_mask(_lib.ptr(mask), mask.shape[1], n, bx, by, bz, _lib.ptr(st), pitch,
                                 _lib.stream_handle()), "x")
g1 = st[:, :bx * by * bz].view(n, bx, by, bz // 32, 32)
res = {}
# y-pass tiles: (p, x, zblock) over all y
t_max = g1.amax(dim=(2, 4)); t_min = g1.amin(dim=(2, 4))
res["y_tiles_all255"] = float(((t_min == 255)).float().mean())
res["y_tiles_all0"] = float(((t_max == 0)).float().mean())
# x-pass tiles (64 z of one (p, y) over all x), before pass x: x-line has no occupied block
# -> after pass x all 255
g1x = st[:, :bx * by * bz].view(n, bx, by, bz // 64, 64)
res["x_tiles_all255_after"] = float((g1x.amin(dim=(1, 4)) == 255).float().mean())
res["x_tiles_all0_after"] = float((g1x.amax(dim=(1, 4)) == 0).float().mean())
pset = pdm.build_pdm_set(vol, grid, scheme, cfg["mode"])
f = pset.storage[:, :bx * by * bz].view(n, bx * by // 32, 32 * bz)
res["z_tiles_all255"] = float((f.amin(dim=2) == 255).float().mean())
res["z_tiles_all0"] = float((f.amax(dim=2) == 0).float().mean())
per_p = ((g1.amin(dim=(2, 4)) == 255) | (g1.amax(dim=(2, 4)) == 0)).float().mean(dim=(1, 2))
res["y_const_by_partition"] = [round(float(v), 3) for v in per_p]
print(json.dumps(res))
