"""Config c, a few TF-change merges of the bench's TF sequence (for ncu):
build the PDM set, then select + combine_flags_into for timed steps with
k = 8, 16, 29 (argv overrides), one launch each, in that order."""
import sys
from pathlib import Path

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
_, timed = bench.tf_plan(cfg["n"], cfg["bits"], 32, 5, cfg["seed"] + 1)
ks = [int(a) for a in sys.argv[1:]] or [8, 16, 29]
out = torch.empty(grid.bdims, dtype=torch.uint8, device="cuda")
flags = torch.empty(cfg["n"], dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k in ks:
    picks, alpha = timed[k - 1]
    a = torch.from_numpy(alpha).cuda()
    flush.fill_(k)
    pdm.select_partitions_device(a, scheme, flags)
    pdm.acceleration.combine_flags_into(pset, flags, out)
torch.cuda.synchronize()
print("ok", ks)
