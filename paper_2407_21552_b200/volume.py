"""Volumes and block geometry (drop-in for pdmrender.volume's hot-path names).

Mirrors /root/reference/pkg/src/pdmrender/volume.py: ``BlockGrid`` (:33-62),
``Volume`` (:65-116), ``load_raw``/``save_raw`` (:119-178) and
``block_min_max`` (:289-300) with the same arguments, defaults, layouts and
exceptions.  Differences are B200-side only:

* a ``Volume`` can also be device-born (``Volume.from_device``): its voxels
  live in HBM and are downloaded only if ``.voxels`` is read; its
  ``intensity_range`` comes from a device reduction;
* ``Volume.device_voxels()`` uploads host voxels once and caches them, so the
  block-reduction kernels never re-copy a volume;
* ``block_min_max`` runs the apron min/max kernel and returns host arrays
  (reference contract); ``block_min_max_device`` keeps them in HBM.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib, device

_DTYPES = {8: np.uint8, 16: np.uint16}


class VolumeError(ValueError):
    """Invalid volume data or metadata."""


class SizeMismatchError(VolumeError):
    """RAW payload length disagrees with dims x bytes per voxel."""


class BitDepthError(VolumeError):
    """A bit depth other than 8 or 16."""


@dataclass(frozen=True)
class BlockGrid:
    """Non-overlapping b^3 blocks covering a volume; edge blocks may be partial
    (bdims = ceil(dims / b), volume.py:33-53)."""

    b: int
    dims: tuple[int, int, int]
    bdims: tuple[int, int, int]

    @classmethod
    def for_dims(cls, dims, b: int = 4) -> "BlockGrid":
        if b < 1:
            raise ValueError(f"block edge must be >= 1, got {b}")
        d = tuple(int(v) for v in dims)
        if len(d) != 3 or min(d) < 1:
            raise ValueError(f"dims must be three positive integers, got {d}")
        return cls(b=int(b), dims=d, bdims=tuple((v + b - 1) // b for v in d))

    @property
    def num_blocks(self) -> int:
        return self.bdims[0] * self.bdims[1] * self.bdims[2]

    def block_of(self, voxel) -> tuple[int, int, int]:
        return tuple(int(v) // self.b for v in voxel)


class Volume:
    """A uint8/uint16 scalar volume indexed [x, y, z] (z contiguous), its
    spacing and attained intensity range (volume.py:65-116)."""

    __slots__ = ("dims", "spacing", "intensity_range", "_host", "_dev", "_bits")

    def __init__(self, dims, voxels, spacing=(1.0, 1.0, 1.0)):
        if not isinstance(voxels, np.ndarray):
            raise VolumeError("Volume(voxels=...) takes a host numpy array; "
                              "use Volume.from_device for device-born volumes")
        if voxels.dtype not in (np.uint8, np.uint16):
            raise BitDepthError(f"unsupported voxel dtype {voxels.dtype}")
        d = tuple(int(v) for v in dims)
        if voxels.shape != d:
            raise VolumeError(f"voxel array shape {voxels.shape} does not match dims {d}")
        self._init_common(d, spacing, 8 if voxels.dtype == np.uint8 else 16)
        self._host = voxels
        self._dev = None
        self.intensity_range = (int(voxels.min()), int(voxels.max()))

    def _init_common(self, dims, spacing, bits):
        sp = tuple(float(s) for s in spacing)
        if any(s <= 0 for s in sp):
            raise VolumeError(f"spacing must be positive, got {spacing}")
        self.dims = dims
        self.spacing = sp
        self._bits = bits

    # -- constructors ---------------------------------------------------------
    @classmethod
    def from_array(cls, voxels: np.ndarray, spacing=(1.0, 1.0, 1.0)) -> "Volume":
        voxels = np.ascontiguousarray(voxels)
        return cls(dims=tuple(voxels.shape), voxels=voxels, spacing=spacing)

    @classmethod
    def from_device(cls, voxels_dev, bits: int, dims=None, spacing=(1.0, 1.0, 1.0),
                    intensity_range=None) -> "Volume":
        """Wrap a CUDA tensor holding C-order [x][y][z] voxels (uint8, or int16
        holding uint16 bit patterns).  The host copy is made only on demand."""
        if bits not in _DTYPES:
            raise BitDepthError(f"unsupported bit depth {bits}")
        self = cls.__new__(cls)
        d = tuple(int(v) for v in (dims if dims is not None else voxels_dev.shape))
        if tuple(voxels_dev.shape) != d:
            raise VolumeError(f"device voxels shape {tuple(voxels_dev.shape)} != dims {d}")
        if voxels_dev.element_size() * 8 != bits or not voxels_dev.is_cuda:
            raise VolumeError("device voxels must be a CUDA tensor of the volume's bit depth")
        self._init_common(d, spacing, bits)
        self._host = None
        self._dev = voxels_dev.contiguous()
        if intensity_range is None:
            intensity_range = _device_range(self._dev, bits)
        self.intensity_range = tuple(int(v) for v in intensity_range)
        return self

    # -- properties -----------------------------------------------------------
    @property
    def voxels(self) -> np.ndarray:
        if self._host is None:
            self._host = device.to_host(self._dev, _DTYPES[self._bits])
        return self._host

    @property
    def bits(self) -> int:
        return self._bits

    @property
    def dtype(self):
        return np.dtype(_DTYPES[self._bits])

    @property
    def num_voxels(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    @property
    def nbytes(self) -> int:
        return self.num_voxels * (self._bits // 8)

    def device_voxels(self):
        """The voxels in HBM (uploaded on first use, then cached)."""
        if self._dev is None:
            self._dev = device.to_device(self._host)
        return self._dev

    def histogram(self, bins: int = 256) -> np.ndarray:
        """Fixed-width histogram over the representable range (volume.py:110-116)."""
        shift = self.bits - int(round(math.log2(bins)))
        if shift < 0:
            raise ValueError(f"cannot split {self.bits}-bit range into {bins} bins")
        v = self.voxels
        coarse = v >> shift if shift else v
        return np.bincount(coarse.ravel().astype(np.int64), minlength=bins)

    def __repr__(self) -> str:
        where = "device" if self._host is None else "host"
        return f"Volume(dims={self.dims}, bits={self.bits}, {where})"


def _device_range(voxels_dev, bits):
    """(min, max) of device voxels via the pdm_volume_range reduction kernel."""
    L = _lib.lib()
    out = device.empty((2,), np.int32)
    _lib.check(L.pdm_volume_range(_lib.ptr(voxels_dev), bits, voxels_dev.numel(), _lib.ptr(out),
                                  _lib.stream_handle()), "pdm_volume_range")
    lo, hi = device.to_host(out, np.int32).tolist()
    return int(lo), int(hi)


def load_raw(data_path, meta_path) -> Volume:
    """RAW (x-fastest) + JSON metadata loader (volume.py:119-161)."""
    meta_path, data_path = Path(meta_path), Path(data_path)
    try:
        meta = json.loads(meta_path.read_text())
    except json.JSONDecodeError as exc:
        raise VolumeError(f"malformed metadata JSON in {meta_path}: {exc}") from exc
    missing = [k for k in ("dims", "bits") if k not in meta]
    if missing:
        raise VolumeError(f"metadata {meta_path} is missing required key {missing[0]!r}")
    dims = tuple(int(d) for d in meta["dims"])
    if len(dims) != 3 or min(dims) < 1:
        raise VolumeError(f"metadata dims must be three positive integers, got {dims}")
    bits = int(meta["bits"])
    if bits not in _DTYPES:
        raise BitDepthError(f"unsupported bit depth {bits} (expected 8 or 16)")
    endian = meta.get("endianness", "le")
    if endian not in ("le", "be"):
        raise VolumeError(f"unsupported endianness {endian!r}")
    spacing = tuple(float(s) for s in meta.get("spacing", (1.0, 1.0, 1.0)))
    raw = data_path.read_bytes()
    want = dims[0] * dims[1] * dims[2] * (bits // 8)
    if len(raw) != want:
        raise SizeMismatchError(
            f"{data_path} holds {len(raw)} bytes, expected {want} for dims {dims} at {bits} bits")
    src_dtype = np.dtype(np.uint8) if bits == 8 else np.dtype("<u2" if endian == "le" else ">u2")
    flat = np.frombuffer(raw, dtype=src_dtype).astype(_DTYPES[bits])
    # x-fastest on disk == Fortran order for [x, y, z]; store C-order (z contiguous)
    vox = np.ascontiguousarray(flat.reshape(dims, order="F"))
    return Volume(dims=dims, voxels=vox, spacing=spacing)


def save_raw(volume: Volume, data_path, meta_path) -> None:
    """Little-endian x-fastest RAW + JSON (volume.py:164-178)."""
    flat = volume.voxels.flatten(order="F")
    if volume.bits == 16:
        flat = flat.astype("<u2")
    Path(data_path).write_bytes(flat.tobytes())
    meta = {"dims": list(volume.dims), "bits": volume.bits, "endianness": "le",
            "spacing": list(volume.spacing)}
    Path(meta_path).write_text(json.dumps(meta, indent=2) + "\n")


def check_pair(volume: Volume, grid: BlockGrid) -> None:
    if tuple(grid.dims) != tuple(volume.dims):
        raise VolumeError(f"grid dims {grid.dims} do not match volume dims {volume.dims}")


def block_min_max_device(volume: Volume, grid: BlockGrid):
    """Apron min/max per block as CUDA tensors (volume dtype bit patterns)."""
    check_pair(volume, grid)
    L = _lib.lib()
    vox = volume.device_voxels()
    mins = device.empty(grid.bdims, volume.dtype)
    maxs = device.empty(grid.bdims, volume.dtype)
    _lib.check(L.pdm_block_min_max(_lib.ptr(vox), volume.bits, *volume.dims, grid.b,
                                   _lib.ptr(mins), _lib.ptr(maxs), _lib.stream_handle()),
               "pdm_block_min_max")
    return mins, maxs


def block_min_max(volume: Volume, grid: BlockGrid) -> tuple[np.ndarray, np.ndarray]:
    """Per-block min/max over the block grown by a clipped 1-voxel apron
    (volume.py:289-300); host arrays of the volume's dtype, shape bdims."""
    mins, maxs = block_min_max_device(volume, grid)
    return device.to_host(mins, volume.dtype), device.to_host(maxs, volume.dtype)
