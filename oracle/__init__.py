"""CPU oracle for the distance-map update path -- TEST INFRASTRUCTURE ONLY.

This package restates the reference's hot path (``pdmrender`` in
/root/reference/pkg/src) over numpy arrays by calling the C restatement in
``pdm_oracle.c``.  It is the checker the CUDA path is compared against and the
CPU baseline bench.py times.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import it;
the product package ``paper_2407_21552_b200`` never does.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``), so parity is pinned, not assumed.

Each wrapper names the reference function it restates (file:line relative to
/root/reference/pkg/src/pdmrender).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle_pdm.so"
_lib = None

_I64 = ctypes.c_int64
_P = ctypes.c_void_p


def build(force: bool = False) -> Path:
    """Compile pdm_oracle.c with the committed Makefile (gcc, OpenMP)."""
    newest = max((_HERE / f).stat().st_mtime for f in ("pdm_oracle.c", "march_oracle.c",
                                                        "Makefile"))
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < newest:
        subprocess.run(["make", "-C", str(_HERE), "-B" if force else "-s"], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        sig = {
            "oracle_set_threads": (None, [ctypes.c_int]),
            "oracle_max_threads": (ctypes.c_int, []),
            "oracle_chamfer_chebyshev": (None, [_P, _I64, _I64, _I64, _P]),
            "oracle_distance_transform": (ctypes.c_int, [_P, _I64, _I64, _I64, _P]),
            "oracle_distance_transform_batch": (ctypes.c_int, [_P, _I64, _I64, _I64, _I64, _P]),
            "oracle_partition_presence": (None, [_P, ctypes.c_int, _I64, _I64, _I64, _I64, _P, _I64, _P]),
            "oracle_block_any_in_range": (
                None, [_P, ctypes.c_int, _I64, _I64, _I64, _I64, ctypes.c_uint32, ctypes.c_uint32, _P]),
            "oracle_block_any_nonzero": (None, [_P, ctypes.c_int, _I64, _I64, _I64, _I64, _P, _P]),
            "oracle_block_min_max": (None, [_P, ctypes.c_int, _I64, _I64, _I64, _I64, _P, _P]),
            "oracle_range_apron_presence": (None, [_P, _P, ctypes.c_int, _I64, _P, _P, _I64, _P]),
            "oracle_range_apron_tf": (ctypes.c_int, [_P, _P, ctypes.c_int, _I64, _P, _I64, _I64, _P]),
            "oracle_select": (None, [_P, _I64, _I64, _P, _I64, _P]),
            "oracle_combine": (None, [_P, _I64, _P, _I64, _P]),
            "oracle_march_rays": (None, [_P, ctypes.c_int, _I64, _I64, _I64, _P, _I64, _P, _I64,
                                         ctypes.c_double, ctypes.c_int, ctypes.c_double, _P, _P,
                                         _I64, _P, _P]),
            "oracle_synth_volume": (
                None, [ctypes.c_int, _I64, _I64, _I64, _I64, _I64, _P, _I64, ctypes.c_uint64, _P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        set_threads(int(os.environ.get("ORACLE_THREADS", "1")))
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data


def _bits(vox: np.ndarray) -> int:
    if vox.dtype == np.uint8:
        return 8
    if vox.dtype == np.uint16:
        return 16
    raise TypeError(f"unsupported voxel dtype {vox.dtype}")


def _bdims(dims, b):
    return tuple(-(-int(d) // int(b)) for d in dims)


# --- L0 kernels ---------------------------------------------------------------

def chamfer_chebyshev(occ: np.ndarray) -> np.ndarray:
    """_kernels.py:17-81 -- int32 chessboard distance, INF32 = 1<<20 when empty."""
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    out = np.empty(occ.shape, dtype=np.int32)
    lib().oracle_chamfer_chebyshev(_ptr(occ), *occ.shape, _ptr(out))
    return out


def distance_transform(occ: np.ndarray) -> np.ndarray:
    """acceleration.py:177-181 -- uint8 distance map clamped at 255."""
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    out = np.empty(occ.shape, dtype=np.uint8)
    if lib().oracle_distance_transform(_ptr(occ), *occ.shape, _ptr(out)):
        raise MemoryError("oracle distance transform allocation failed")
    return out


def distance_transform_batch(occs: np.ndarray) -> np.ndarray:
    """acceleration.py:230-233 -- one distance transform per partition [n, bx, by, bz]."""
    occs = np.ascontiguousarray(occs, dtype=np.uint8)
    out = np.empty(occs.shape, dtype=np.uint8)
    if lib().oracle_distance_transform_batch(_ptr(occs), *occs.shape, _ptr(out)):
        raise MemoryError("oracle distance transform allocation failed")
    return out


def partition_presence(vox: np.ndarray, b: int, pid: np.ndarray, n: int) -> np.ndarray:
    """_kernels.py:137-149 -- bool [n, bx, by, bz] presence of each partition per block."""
    vox = np.ascontiguousarray(vox)
    pid = np.ascontiguousarray(pid, dtype=np.int32)
    out = np.zeros((n,) + _bdims(vox.shape, b), dtype=np.uint8)
    lib().oracle_partition_presence(_ptr(vox), _bits(vox), *vox.shape, b, _ptr(pid), n, _ptr(out))
    return out.astype(bool)


def block_any_in_range(vox: np.ndarray, b: int, lo: int, hi: int) -> np.ndarray:
    """_kernels.py:84-110."""
    vox = np.ascontiguousarray(vox)
    out = np.empty(_bdims(vox.shape, b), dtype=np.uint8)
    lib().oracle_block_any_in_range(_ptr(vox), _bits(vox), *vox.shape, b, lo, hi, _ptr(out))
    return out.astype(bool)


def block_any_nonzero(vox: np.ndarray, b: int, nz_lut: np.ndarray) -> np.ndarray:
    """_kernels.py:113-134."""
    vox = np.ascontiguousarray(vox)
    nz_lut = np.ascontiguousarray(nz_lut, dtype=np.uint8)
    out = np.empty(_bdims(vox.shape, b), dtype=np.uint8)
    lib().oracle_block_any_nonzero(_ptr(vox), _bits(vox), *vox.shape, b, _ptr(nz_lut), _ptr(out))
    return out.astype(bool)


def block_min_max(vox: np.ndarray, b: int) -> tuple[np.ndarray, np.ndarray]:
    """volume.py:262-300 -- apron (1 voxel, clipped) min/max per block, volume dtype."""
    vox = np.ascontiguousarray(vox)
    bd = _bdims(vox.shape, b)
    mins = np.empty(bd, dtype=vox.dtype)
    maxs = np.empty(bd, dtype=vox.dtype)
    lib().oracle_block_min_max(_ptr(vox), _bits(vox), *vox.shape, b, _ptr(mins), _ptr(maxs))
    return mins, maxs


# --- L1 functions (acceleration.py / transfer.py) ---------------------------

def pid_lut(bounds) -> np.ndarray:
    """transfer.py:168-171 -- 0-based partition index per intensity."""
    widths = [hi - lo + 1 for lo, hi in bounds]
    return np.repeat(np.arange(len(bounds), dtype=np.int32), widths)


def range_apron_presence(mins, maxs, bounds) -> np.ndarray:
    """acceleration.py:223-229 (and :138-141 for one partition)."""
    mins = np.ascontiguousarray(mins)
    maxs = np.ascontiguousarray(maxs)
    lo = np.array([p[0] for p in bounds], dtype=np.uint32)
    hi = np.array([p[1] for p in bounds], dtype=np.uint32)
    out = np.empty((len(bounds),) + mins.shape, dtype=np.uint8)
    lib().oracle_range_apron_presence(_ptr(mins), _ptr(maxs), _bits(mins), mins.size,
                                      _ptr(lo), _ptr(hi), len(bounds), _ptr(out))
    return out.astype(bool)


def occupancy_for_partition(vox, b, lo, hi, mode="voxel", minmax=None) -> np.ndarray:
    """acceleration.py:114-142."""
    if mode == "voxel":
        return block_any_in_range(vox, b, lo, hi)
    mins, maxs = minmax if minmax is not None else block_min_max(vox, b)
    return range_apron_presence(mins, maxs, [(lo, hi)])[0]


def occupancy_for_tf(vox, b, lut: np.ndarray, mode="voxel", minmax=None) -> np.ndarray:
    """acceleration.py:145-174."""
    alpha = np.ascontiguousarray(np.asarray(lut, dtype=np.float64)[:, 3])
    if mode == "voxel":
        return block_any_nonzero(vox, b, (alpha > 0.0).astype(np.uint8))
    mins, maxs = minmax if minmax is not None else block_min_max(vox, b)
    mins = np.ascontiguousarray(mins)
    maxs = np.ascontiguousarray(maxs)
    out = np.empty(mins.shape, dtype=np.uint8)
    lib().oracle_range_apron_tf(_ptr(mins), _ptr(maxs), _bits(mins), mins.size,
                                _ptr(alpha), alpha.size, 1, _ptr(out))
    return out.astype(bool)


def standard_distance_map(vox, b, lut, mode="voxel", minmax=None) -> np.ndarray:
    """acceleration.py:184-196 -- the full recompute for one TF."""
    return distance_transform(occupancy_for_tf(vox, b, lut, mode, minmax))


def build_pdm_set(vox, b, bounds, mode="range_apron") -> np.ndarray:
    """acceleration.py:199-241 -- uint8 [n, bx, by, bz] partitioned distance maps."""
    if mode == "voxel":
        occs = partition_presence(vox, b, pid_lut(bounds), len(bounds))
    else:
        mins, maxs = block_min_max(vox, b)
        occs = range_apron_presence(mins, maxs, bounds)
    return distance_transform_batch(occs)


def select(alpha: np.ndarray, bounds) -> list[int]:
    """transfer.py:250-259 -- sorted 1-based selected partitions."""
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    pid = pid_lut(bounds)
    flags = np.empty(len(bounds), dtype=np.uint8)
    lib().oracle_select(_ptr(alpha), alpha.size, 1, _ptr(pid), len(bounds), _ptr(flags))
    return [int(i) + 1 for i in np.flatnonzero(flags)]


def combine(pdms: np.ndarray, selected_1based, out: np.ndarray | None = None) -> np.ndarray:
    """acceleration.py:244-276 -- min over the selected maps, all-255 when empty."""
    pdms = np.ascontiguousarray(pdms, dtype=np.uint8)
    sel = np.ascontiguousarray(sorted(int(i) - 1 for i in selected_1based), dtype=np.int32)
    if out is None:
        out = np.empty(pdms.shape[1:], dtype=np.uint8)
    map_bytes = int(np.prod(pdms.shape[1:]))
    lib().oracle_combine(_ptr(pdms), map_bytes, _ptr(sel), sel.size, _ptr(out))
    return out


def synth_volume(bits: int, dims, boxes: np.ndarray, seed: int, x_range=None) -> np.ndarray:
    """The shared hash-box generator (see pdm_oracle.c); x_range selects a slab."""
    nx, ny, nz = (int(d) for d in dims)
    xs0, xs1 = (0, nx) if x_range is None else (int(x_range[0]), int(x_range[1]))
    boxes = np.ascontiguousarray(boxes, dtype=np.int64).reshape(-1, 8)
    out = np.empty((xs1 - xs0, ny, nz), dtype=np.uint8 if bits == 8 else np.uint16)
    lib().oracle_synth_volume(bits, nx, ny, nz, xs0, xs1, _ptr(boxes), boxes.shape[0],
                              ctypes.c_uint64(seed), _ptr(out))
    return out


def build_pdm_set_synth(bits: int, dims, boxes: np.ndarray, seed: int, b: int, bounds,
                        mode: str = "range_apron", slab_voxels: int = 256) -> np.ndarray:
    """acceleration.py:199-241 on the shared hash-box volume, generated and
    reduced one x-slab at a time so a 2048^3 volume (17 GB) is never held
    whole: each slab's block occupancy is computed on the slab grown by one
    block per side (range_apron: the 1-voxel apron of the slab's edge blocks
    lies in the neighbour slab; block_min_max clips only at the real volume
    ends, volume.py:289-300), stitched into [n, bx, by, bz], then the
    per-partition distance transforms run on the whole grid.  Identical to
    build_pdm_set(synth_volume(...)) -- tested at small sizes."""
    nx = int(dims[0])
    n = len(bounds)
    bd = _bdims(dims, b)
    occs = np.zeros((n,) + bd, dtype=np.uint8)
    step = max(b, (int(slab_voxels) // b) * b)
    pid = pid_lut(bounds)
    for x0 in range(0, nx, step):
        x1 = min(nx, x0 + step)
        bx0, bx1 = x0 // b, -(-x1 // b)
        if mode == "voxel":
            vox = synth_volume(bits, dims, boxes, seed, x_range=(x0, x1))
            occs[:, bx0:bx1] = partition_presence(vox, b, pid, n)
        else:
            lo, hi = max(0, x0 - b), min(nx, x1 + b)
            vox = synth_volume(bits, dims, boxes, seed, x_range=(lo, hi))
            mins, maxs = block_min_max(vox, b)
            off = (x0 - lo) // b
            occs[:, bx0:bx1] = range_apron_presence(mins[off:off + bx1 - bx0],
                                                    maxs[off:off + bx1 - bx0], bounds)
        del vox
    return distance_transform_batch(occs)


def march_rays(vox, lut, dist, b, step, ert_on, ert_thr, origin, dirs):
    """_kernels.py:206-365 -- (rgba float64 [n, 4], counters int64 [n, 4])."""
    vox = np.ascontiguousarray(vox)
    lut = np.ascontiguousarray(lut, dtype=np.float64)
    dist = np.ascontiguousarray(dist, dtype=np.uint8)
    origin = np.ascontiguousarray(origin, dtype=np.float64)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    n = dirs.shape[0]
    rgba = np.empty((n, 4), np.float64)
    counters = np.empty((n, 4), np.int64)
    lib().oracle_march_rays(_ptr(vox), _bits(vox), *vox.shape, _ptr(lut), lut.shape[0],
                            _ptr(dist), int(b), float(step), int(bool(ert_on)), float(ert_thr),
                            _ptr(origin), _ptr(dirs), n, _ptr(rgba), _ptr(counters))
    return rgba, counters
