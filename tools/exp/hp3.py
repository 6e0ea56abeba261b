"""D'-to-host pipeline pieces at config c: kernel-only (pieces=1 minus host
decode is not separable, so: total per format/pieces, and host decode alone)."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2407_21552_b200 as pdm  # noqa: E402
from paper_2407_21552_b200 import _lib, synth  # noqa: E402

L = _lib.lib()
vol = synth.synth_volume_device((1024, 1024, 1024), 16, seed=2407, nbox=12)
grid = pdm.BlockGrid.for_dims(vol.dims, 4)
scheme = pdm.scheme_uniform(32, 16)
pset = pdm.build_pdm_set(vol, grid, scheme)
nib, nib_pitch, base, base_pitch = pset.packed()
nib_h, base_h = pset._host_stage()
nb = grid.num_blocks
out = np.empty(nb, np.uint8)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = _lib.stream_handle()


def timed(fn, reps=20):
    ts = []
    for r in range(reps + 3):
        flush.fill_(r & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append((time.perf_counter() - t0) * 1e3)
    return round(float(np.median(ts)), 4)


res = {}
rng = np.random.default_rng(5)
for k in (1, 4, 16, 28):
    sel = np.ascontiguousarray(np.sort(rng.choice(32, k, replace=False)), dtype=np.int32)
    for fmt in (2, 3):
        for pieces in (1, 4):
            res[f"k{k}_f{fmt}_p{pieces}"] = timed(lambda: L.pdm_merge_packed_to_host(
                _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, None, nb, 32, None,
                sel.ctypes.data, k, _lib.ptr(nib_h), _lib.ptr(base_h), out.ctypes.data, pieces,
                fmt, st))
        if fmt == 2:
            res[f"k{k}_unpack_delta"] = timed(lambda: L.pdm_unpack_delta_host(
                _lib.ptr(nib_h), _lib.ptr(base_h), nb, out.ctypes.data))
        else:
            res[f"k{k}_unpack_sparse"] = timed(lambda: L.pdm_unpack_sparse_host(
                _lib.ptr(nib_h), nb, out.ctypes.data))
    want = torch.stack([pset.storage[i, :nb] for i in sel]).min(0).values.cpu().numpy()
    res[f"k{k}_exact"] = bool(np.array_equal(out, want))
print(json.dumps(res))

# public-API e2e per step (bench sequence), per format
import os  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402

seq = bench.tf_sequence(32, 1 << 16, 36, 2408)
tfs = []
for k, a in seq:
    lut = np.zeros((1 << 16, 4))
    lut[:, 3] = a
    tfs.append((k, pdm.TransferFunction(lut=lut)))
per = {}
for fmt in ("2", "3", "2", "3"):
    os.environ["PDM_HOST_FORMAT"] = fmt
    for i, (k, tf) in enumerate(tfs):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = pdm.combine(pset, pdm.select_partitions(tf, scheme)).dist
        t1 = time.perf_counter()
        if i >= 4:
            per.setdefault(fmt, {}).setdefault(k, []).append(round((t1 - t0) * 1e3, 3))
print(json.dumps({f: {k: min(v) for k, v in sorted(d.items())} for f, d in per.items()}))
print(json.dumps({f: round(float(np.mean([np.mean(v) for v in d.values()])), 4) for f, d in per.items()}))
