"""PDM_HOST_TRACE timeline of pdm_merge_packed_to_host (format 3, 1/4 pieces)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402
import paper_2407_21552_b200 as pdm  # noqa: E402
from paper_2407_21552_b200 import _lib, synth, device  # noqa: E402

L = _lib.lib()
vol = synth.synth_volume_device((1024, 1024, 1024), 16, seed=2407, nbox=12)
grid = pdm.BlockGrid.for_dims(vol.dims, 4)
pset = pdm.build_pdm_set(vol, grid, pdm.scheme_uniform(32, 16))
nib, nib_pitch, base, base_pitch = pset.packed()
nib_h, base_h = pset._host_stage()
nb = grid.num_blocks
sel = np.ascontiguousarray(np.arange(0, 32, 2), dtype=np.int32)
out = device.host_buffer((nb,))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = _lib.stream_handle()
for pieces in (1, 4, 1, 4):
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.pdm_merge_packed_to_host(_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, None, nb, 32,
                               None, sel.ctypes.data, 16, _lib.ptr(nib_h), _lib.ptr(base_h),
                               out.ctypes.data, pieces, 3, st)
    print(f"pieces={pieces} total {(time.perf_counter() - t0) * 1e6:.1f} us", file=sys.stderr,
          flush=True)
