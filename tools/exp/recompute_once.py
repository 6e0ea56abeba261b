"""Three standard_distance_map calls per mode at config c (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

import paper_2407_21552_b200 as pdm  # noqa: E402
from paper_2407_21552_b200 import synth  # noqa: E402

vol = synth.synth_volume_device((1024, 1024, 1024), 16, seed=2407, nbox=12)
grid = pdm.BlockGrid.for_dims(vol.dims, 4)
tf = pdm.tf_archetype("tf3", 16)
mm = pdm.block_min_max_device(vol, grid)
for _ in range(3):
    for m in ("voxel", "range_apron"):
        pdm.standard_distance_map(vol, grid, tf, m, minmax=mm if m == "range_apron" else None)
torch.cuda.synchronize()
