"""Seeded synthetic volumes with the statistics of the reference's
``random_structured_volume`` (/root/reference/pkg/tests/conftest.py:59-78):
background 0 plus a few axis-aligned boxes, each filled with intensities from
its own band, so per-partition occupancy varies (uniform noise would make
every block occupied for every partition).

Large volumes are generated on the device by ``pdm_synth_volume`` from the
box table built here; the CPU oracle evaluates the identical per-voxel hash
(oracle_synth_volume), so both arms see the same bytes.
"""

from __future__ import annotations

import numpy as np

from . import _lib, device
from .volume import Volume


def synth_boxes(dims, bits: int, seed: int, nbox: int = 12) -> np.ndarray:
    """int64 [nbox, 8] table: x0 x1 y0 y1 z0 z1 band_lo band_hi."""
    rng = np.random.default_rng(seed)
    span = 1 << bits
    rows = []
    for _ in range(nbox):
        row = []
        for d in dims:
            size = max(1, int(d * rng.uniform(0.08, 0.45)))
            lo = int(rng.integers(0, max(1, d - size)))
            row += [lo, min(d, lo + size)]
        band_lo = int(rng.integers(1, span))
        band_hi = min(span - 1, band_lo + int(rng.integers(0, max(2, span // 8))))
        rows.append(row + [band_lo, band_hi])
    return np.asarray(rows, dtype=np.int64)


def synth_volume_device(dims, bits: int, seed: int = 0, nbox: int = 12, x_range=None) -> Volume:
    """Device-born synthetic volume (or an x-slab [x0, x1) of it)."""
    L = _lib.lib()
    nx, ny, nz = (int(d) for d in dims)
    x0, x1 = (0, nx) if x_range is None else (int(x_range[0]), int(x_range[1]))
    boxes = np.ascontiguousarray(synth_boxes((nx, ny, nz), bits, seed, nbox))
    out = device.empty((x1 - x0, ny, nz), np.uint8 if bits == 8 else np.uint16)
    _lib.check(L.pdm_synth_volume(bits, nx, ny, nz, x0, x1, boxes.ctypes.data, boxes.shape[0],
                                  seed, _lib.ptr(out), _lib.stream_handle()), "pdm_synth_volume")
    return Volume.from_device(out, bits)
