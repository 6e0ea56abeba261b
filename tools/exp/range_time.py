"""pdm_volume_range at config c (1024^3 u16) and 256^3 u8, CUDA events."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402
from paper_2407_21552_b200 import _lib  # noqa: E402

L = _lib.lib()
for bits, n in ((16, 1 << 30), (8, 1 << 24)):
    v = torch.randint(0, 1 << bits, (n,), dtype=torch.int32, device="cuda").to(
        torch.uint8 if bits == 8 else torch.int16)
    out = torch.empty(2, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.pdm_volume_range(_lib.ptr(v), bits, n, _lib.ptr(out), _lib.stream_handle())
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"bits={bits} voxels={n} {ms:.4f} ms = {v.numel() * v.element_size() / ms / 1e6:.0f} GB/s")
