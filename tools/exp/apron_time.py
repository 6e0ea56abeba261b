"""range_apron partition mask and block min/max at a cube of side argv[1]
(u16, b=4, n=32), CUDA events, min of 5 (A/B of apron kernel settings)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

import paper_2407_21552_b200 as pdm  # noqa: E402
from paper_2407_21552_b200 import synth  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
vol = synth.synth_volume_device((side,) * 3, 16, seed=2407, nbox=12)
grid = pdm.BlockGrid.for_dims(vol.dims, 4)
scheme = pdm.scheme_uniform(32, 16)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(min(ts), 4)


pdm.partition_mask(vol, grid, scheme, "range_apron")
r = {"side": side, "mask_range_apron_ms": timed(lambda: pdm.partition_mask(vol, grid, scheme, "range_apron")),
     "block_min_max_ms": timed(lambda: pdm.block_min_max_device(vol, grid))}
r["GBps"] = round(vol.nbytes / r["mask_range_apron_ms"] / 1e6, 1)
print(json.dumps(r))
