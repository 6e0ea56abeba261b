"""Config c: one build_pdm_set (range_apron) after a warm-up build -- for ncu
captures of the precompute kernels (apron POM, expand, DT passes, packing)."""
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
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    pset = pdm.build_pdm_set(vol, grid, scheme, cfg["mode"])
torch.cuda.synchronize()
print("ok")
