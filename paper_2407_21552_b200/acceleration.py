"""Partitioned occupancy / distance maps on B200 -- the distance-map update path.

Drop-in for /root/reference/pkg/src/pdmrender/acceleration.py: the same
public names, signatures, defaults, validation order and exceptions
(``OccupancyMap``/``DistanceMap``/``PdmSet`` :42-99, ``occupancy_for_partition``
:114-142, ``occupancy_for_tf`` :145-174, ``distance_transform`` :177-181,
``standard_distance_map`` :184-196, ``build_pdm_set`` :199-241, ``combine``
:244-276, dumps :279-354).  Every computation runs in libpdm_b200 kernels:

  K1/K2  pdm_partition_mask_voxel / pdm_partition_mask_range_apron  (POM build)
  K3-K5  pdm_block_any_lut / pdm_occupancy_minmax_{range,prefix}   (occupancy)
  K6     pdm_distance_transform[_mask]                              (Chebyshev DT)
  K7     pdm_combine / pdm_combine_flags                            (TF-change merge)
  K8     pdm_select                                                 (selection)

Residency: maps live in HBM.  A ``PdmSet`` owns one partition-major
[n][plane_pitch] uint8 allocation; ``DistanceMap``/``OccupancyMap`` hold a CUDA
tensor and download ``.dist`` / ``.occupied`` to numpy on first access
(cached), so callers that read them (raycast, CLI, service) see the reference
types while the update itself never leaves the device.
"""

from __future__ import annotations

import os
import struct
import time
from pathlib import Path

import numpy as np

from . import _lib, device
from .transfer import (
    Partition,
    PartitionScheme,
    PartitionSelection,
    SelectionError,
    TransferFunction,
    alpha_to_device,
    select_partitions_device,
)
from .volume import BlockGrid, Volume, VolumeError, block_min_max_device, check_pair

OCCUPANCY_MODES = ("voxel", "range_apron")
DIST_CLAMP = 255
_MAP_MAGIC = b"PDMD"
_SET_MAGIC = b"PDMS"
_MAX_FLAGS = 4096  # pdm_combine_flags compacts the selection in shared memory
_MAX_PACKED_SEL = 240  # pdm_combine_packed carries the indices in kernel parameters


def _packed_enabled() -> bool:
    # PDM_PACKED=0 keeps the merge on the raw planes (A/B measurements).
    return os.environ.get("PDM_PACKED", "1") != "0"


def _tile_skip_enabled() -> bool:
    # PDM_TILE_SKIP=0: packed merges read every selected plane (A/B).
    return os.environ.get("PDM_TILE_SKIP", "1") != "0"


class OccupancyModeError(ValueError):
    """Unknown occupancy mode string."""


def _require_mode(mode: str) -> None:
    if mode not in OCCUPANCY_MODES:
        raise OccupancyModeError(
            f"unknown occupancy mode {mode!r}; expected one of {OCCUPANCY_MODES}")


class _BlockArray:
    """A per-block array resident on the device, host copy materialised lazily."""

    _np_dtype = np.uint8

    def __init__(self, b, bdims, data, field):
        self.b = int(b)
        self.bdims = tuple(int(v) for v in bdims)
        self._host = None
        self._dev = None
        self._host_fill = None  # fills the host view its own way (compact D' over PCIe)
        shape = tuple(data.shape)
        if shape != self.bdims:
            raise ValueError(f"{field} array shape does not match bdims")
        if isinstance(data, np.ndarray):
            self._host = data
        else:
            self._dev = data

    def _host_array(self):
        if self._host is None:
            if self._host_fill is not None:
                host = device.host_buffer(self.bdims)  # recycled, already faulted in
                self._host_fill(host)
                self._host = host
            else:
                self._host = device.to_host(self.device(), self._np_dtype)
        return self._host

    def device(self):
        """uint8 CUDA tensor of shape bdims (uploaded on first use, then cached)."""
        if self._dev is None:
            self._dev = device.to_device(np.ascontiguousarray(self._host, dtype=np.uint8))
        return self._dev


class OccupancyMap(_BlockArray):
    """One flag per block: True where the block can contribute opacity."""

    _np_dtype = np.bool_

    def __init__(self, b, bdims, occupied):
        super().__init__(b, bdims, occupied, "occupancy")

    @property
    def occupied(self) -> np.ndarray:
        return self._host_array()

    @property
    def occupied_fraction(self) -> float:
        occ = self.occupied
        return float(np.count_nonzero(occ)) / occ.size


class DistanceMap(_BlockArray):
    """Chessboard block distance to the nearest occupied block, clamped at 255
    (0 = occupied, all 255 when nothing is occupied)."""

    def __init__(self, b, bdims, dist):
        super().__init__(b, bdims, dist, "distance")
        if isinstance(dist, np.ndarray) and dist.dtype != np.uint8:
            raise ValueError(f"distance array must be uint8, got {dist.dtype}")
        if not isinstance(dist, np.ndarray) and dist.element_size() != 1:
            raise ValueError("distance tensor must be uint8")

    @classmethod
    def _of_device(cls, b: int, bdims: tuple, t) -> "DistanceMap":
        """A map around a uint8 CUDA tensor of shape bdims that this module
        just made (no validation: the merges' own results)."""
        obj = cls.__new__(cls)
        obj.b = b
        obj.bdims = bdims
        obj._host = None
        obj._dev = t
        obj._host_fill = None
        return obj

    @property
    def dist(self) -> np.ndarray:
        probe = self.__dict__.get("_probe")
        if probe is not None:
            probe.read = True
        return self._host_array()

    @property
    def occupied_fraction(self) -> float:
        """Share of blocks at distance 0 (acceleration.py:77-79); counted on
        the device (8 bytes back) unless the host copy already exists."""
        if self._host is not None:
            d = self._host
            return float(np.count_nonzero(d == 0)) / d.size
        zeros = getattr(self, "_zero_count", None)  # counted by the merge itself
        if zeros is not None:
            return int(zeros.item()) / float(np.prod(self.bdims))
        return count_value(self.device(), 0) / float(np.prod(self.bdims))


def count_value(t_dev, value: int) -> int:
    """Number of bytes of a uint8 CUDA tensor equal to value (pdm_count_value)."""
    L = _lib.lib()
    cnt = device.empty((1,), np.int64)
    _lib.check(L.pdm_count_value(_lib.ptr(t_dev), t_dev.numel(), int(value), _lib.ptr(cnt),
                                 _lib.stream_handle()), "pdm_count_value")
    return int(cnt.item())


class PdmSet:
    """One distance map per partition of a scheme.

    Device layout: ``storage`` is a uint8 CUDA tensor [n, plane_pitch]; map p
    is ``storage[p, :num_blocks]`` viewed as bdims.  ``plane_pitch`` is
    num_blocks rounded up to 256 bytes so every plane is 16-byte aligned for
    the vectorised merge.
    """

    def __init__(self, grid: BlockGrid, scheme: PartitionScheme, pdms=None,
                 occupancy_mode: str = "range_apron", init_seconds: float = 0.0, storage=None):
        self.grid = grid
        self.scheme = scheme
        self.occupancy_mode = occupancy_mode
        self.init_seconds = float(init_seconds)
        self.plane_pitch = device.plane_pitch(grid.num_blocks)
        self._storage = storage
        self._packed = None  # None: not packed yet; False: does not pack; else planes
        self._tile_bounds = None  # per-tile plane bounds of the packed planes
        # every map is a distance field whose z rows hold whole 16-block chunks
        # (built here by the distance transform with bz % 16 == 0): D' can then
        # go to the host in the 5/16-size delta form
        self._delta_ok = False
        if storage is not None:
            nb = grid.num_blocks
            self.pdms = tuple(
                DistanceMap(b=grid.b, bdims=grid.bdims, dist=storage[p, :nb].view(grid.bdims))
                for p in range(storage.shape[0]))
        else:
            self.pdms = tuple(pdms if pdms is not None else ())

    @property
    def n(self) -> int:
        return len(self.pdms)

    def memory_bytes(self) -> int:
        """n * num_blocks (acceleration.py:96-99), excluding plane padding."""
        return self.n * self.grid.num_blocks

    @property
    def storage(self):
        """The [n, plane_pitch] device allocation (assembled on first use when
        the set was built from individual maps)."""
        if self._storage is None:
            nb = self.grid.num_blocks
            st = device.empty((self.n, self.plane_pitch), np.uint8)
            for p, dm in enumerate(self.pdms):
                st[p, :nb].copy_(dm.device().reshape(-1))
            self._storage = st
        return self._storage

    # -- nibble-packed copy of the planes (B200 merge storage) ---------------
    # Every map is a clamped Chebyshev distance field, so 16 consecutive
    # blocks of a z row span <= 15 values and pack losslessly into a base byte
    # plus 4-bit offsets (csrc/packed.cu).  The merge then reads 0.5625 B per
    # block and plane instead of 1 B; results are bit-identical.  The raw
    # storage stays the source of truth: packing runs once (build_pdm_set, or
    # the first merge of a set assembled or loaded otherwise) and is skipped
    # for sets that do not pack (rows of a length not divisible by 16, maps
    # that are not distance fields).  Code that writes into ``storage`` after
    # a merge must call drop_packed().

    def _alloc_packed(self):
        """Device allocations for the packed copy: (nib, nib_pitch, base,
        base_pitch, violation counter)."""
        chunks = int(_lib.lib().pdm_packed_chunks(self.grid.num_blocks))
        nib_pitch = -(-chunks * 8 // 256) * 256
        base_pitch = -(-chunks // 256) * 256
        return (device.empty((self.n, nib_pitch), np.uint8), nib_pitch,
                device.empty((self.n, base_pitch), np.uint8), base_pitch,
                device.empty((1,), np.uint32))

    def _start_pack(self):
        """Launch the packing on the current stream; returns the pending
        state (finished by _finish_pack) or False when disabled/empty."""
        if not _packed_enabled() or self.n == 0:
            return False
        L = _lib.lib()
        planes = self._alloc_packed()
        nib, nib_pitch, base, base_pitch, bad = planes
        _lib.check(L.pdm_pack_pdms(_lib.ptr(self.storage), self.plane_pitch,
                                   self.grid.num_blocks, self.n, _lib.ptr(nib), nib_pitch,
                                   _lib.ptr(base), base_pitch, _lib.ptr(bad),
                                   _lib.stream_handle()), "pdm_pack_pdms")
        return planes

    def _alloc_tile_bounds(self):
        """uint16 [tiles][n] device table for the merge's per-tile plane skip,
        or None when the skip is off (PDM_TILE_SKIP=0)."""
        if not _tile_skip_enabled():
            return None
        return device.empty((-(-self.grid.num_blocks // 1024), self.n), np.int16)

    def _finish_pack(self, pending, tile_bounds=None) -> None:
        """Adopt the packed planes if they packed; tile_bounds: the per-tile
        plane bounds already made with them (the fused z pass), else they are
        computed here (pdm_packed_tile_bounds)."""
        if pending is False:
            self._packed = False
            return
        nib, nib_pitch, base, base_pitch, bad = pending
        ok = int(bad.cpu()[0]) == 0  # int32 view of the uint32 count; 0 either way
        self._packed = (nib, nib_pitch, base, base_pitch) if ok else False
        self._tile_bounds = None
        self._pargs = None
        if ok and tile_bounds is not None:
            self._tile_bounds = tile_bounds
        elif ok and _tile_skip_enabled():
            # per (1024-block tile, plane) min/max: the merges' exact tile skip
            nb = self.grid.num_blocks
            tb = self._alloc_tile_bounds()
            _lib.check(_lib.lib().pdm_packed_tile_bounds(
                _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, nb, self.n, _lib.ptr(tb),
                _lib.stream_handle()), "pdm_packed_tile_bounds")
            self._tile_bounds = tb

    def _packed_args(self):
        """(nib, nib_pitch, base, base_pitch, tile_bounds) as the packed merges
        take them (device pointers), cached; None when the set does not pack."""
        args = self.__dict__.get("_pargs")
        if args is None:
            pk = self.packed()
            if pk is None:
                return None
            nib, nib_pitch, base, base_pitch = pk
            args = self._pargs = (_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                                  self.tile_bounds_ptr())
        return args

    def tile_bounds_ptr(self):
        """Device pointer of the per-tile plane bounds (pdm_packed_tile_bounds)
        of the packed planes, or None."""
        tb = self.__dict__.get("_tile_bounds")
        return _lib.ptr(tb) if tb is not None and self._packed else None

    def packed(self):
        """(nib, nib_pitch, base, base_pitch) device planes, or None when the
        set does not pack (or PDM_PACKED=0)."""
        if self._packed is None:
            self._finish_pack(self._start_pack())
        return self._packed or None

    def _host_stage(self):
        """Pinned host buffers receiving a packed D' (reused across merges;
        each host merge synchronises before returning)."""
        stage = getattr(self, "_stage", None)
        if stage is None:
            t = device.torch()
            chunks = int(_lib.lib().pdm_packed_chunks(self.grid.num_blocks))
            regions = -(-chunks // 64) * 336  # format 3: one 336-byte region per 64 chunks
            stage = (t.empty(max(chunks * 8, regions), dtype=t.uint8, pin_memory=True),
                     t.empty(chunks, dtype=t.uint8, pin_memory=True))
            self._stage = stage
        return stage

    def drop_packed(self) -> None:
        """Forget the packed copy (after writing into ``storage``)."""
        self._packed = None
        self._tile_bounds = None
        self._pargs = None

    def device_bytes(self) -> int:
        """Device bytes held: raw planes plus the packed copy, if any."""
        total = self.n * self.plane_pitch
        pk = self._packed
        if pk:
            total += self.n * (pk[1] + pk[3])
        tb = self.__dict__.get("_tile_bounds")
        if tb is not None:
            total += tb.numel() * 2
        return total


def _mask_words(n: int) -> int:
    return (n + 31) // 32


def occupancy_for_partition(volume: Volume, grid: BlockGrid, partition: Partition,
                            mode: str = "voxel", minmax=None) -> OccupancyMap:
    """Blocks containing (voxel) or possibly reaching (range_apron, 1-voxel
    apron interval test) intensities inside the partition (acceleration.py:114-142)."""
    _require_mode(mode)
    check_pair(volume, grid)
    L = _lib.lib()
    out = device.empty(grid.bdims, np.uint8)
    st = _lib.stream_handle()
    if mode == "voxel":
        lut = np.zeros(1 << volume.bits, dtype=np.uint8)
        lut[partition.rho_lo: partition.rho_hi + 1] = 1
        lut_dev = device.to_device(lut)
        vox = volume.device_voxels()
        _lib.check(L.pdm_block_any_lut(_lib.ptr(vox), volume.bits, *volume.dims, grid.b,
                                       _lib.ptr(lut_dev), _lib.ptr(out), st), "pdm_block_any_lut")
    else:
        mins, maxs = _minmax_device(volume, grid, minmax)
        _lib.check(L.pdm_occupancy_minmax_range(
            _lib.ptr(mins), _lib.ptr(maxs), volume.bits, grid.num_blocks,
            min(partition.rho_lo, 0xFFFFFFFF), min(partition.rho_hi, 0xFFFFFFFF),
            _lib.ptr(out), st), "pdm_occupancy_minmax_range")
    device.complete()
    return OccupancyMap(b=grid.b, bdims=grid.bdims, occupied=out)


def _minmax_device(volume, grid, minmax):
    if minmax is None:
        return block_min_max_device(volume, grid)
    mins, maxs = minmax
    if isinstance(mins, np.ndarray):
        mins = device.to_device(np.ascontiguousarray(mins, dtype=volume.dtype))
        maxs = device.to_device(np.ascontiguousarray(maxs, dtype=volume.dtype))
    if tuple(mins.shape) != tuple(grid.bdims) or tuple(maxs.shape) != tuple(grid.bdims):
        # the reference's OccupancyMap rejects the mis-shaped result
        # (acceleration.py:51-52); here it is caught before any kernel reads
        raise ValueError("occupancy array shape does not match bdims")
    return mins.contiguous(), maxs.contiguous()


def _tf_support(volume: Volume, grid: BlockGrid, tf: TransferFunction, mode: str,
                prefix_too: bool = False):
    """Validation shared by occupancy_for_tf / standard_distance_map
    (acceleration.py:158-163), then the TF's nz LUT and, for range_apron (or
    prefix_too), its prefix count (pdm_alpha_support) on the device."""
    _require_mode(mode)
    check_pair(volume, grid)
    if tf.lut.shape[0] != (1 << volume.bits):
        raise VolumeError(
            f"tf covers {tf.lut.shape[0]} intensities, volume needs {1 << volume.bits}")
    L = _lib.lib()
    span = 1 << volume.bits
    alpha = alpha_to_device(tf)
    nz = device.empty((span,), np.uint8)
    prefix = device.empty((span + 1,), np.int32) if (mode == "range_apron" or prefix_too) \
        else None
    _lib.check(L.pdm_alpha_support(_lib.ptr(alpha), span, 1, _lib.ptr(nz),
                                   _lib.ptr(prefix) if prefix is not None else None,
                                   _lib.stream_handle()), "pdm_alpha_support")
    return nz, prefix


def occupancy_for_tf(volume: Volume, grid: BlockGrid, tf: TransferFunction, mode: str = "voxel",
                     minmax=None) -> OccupancyMap:
    """Blocks that can contribute opacity under a TF (acceleration.py:145-174):
    voxel = any voxel with alpha > 0; range_apron = alpha > 0 somewhere inside
    the block's apron [min, max] (prefix count)."""
    nz, prefix = _tf_support(volume, grid, tf, mode)
    L = _lib.lib()
    st = _lib.stream_handle()
    out = device.empty(grid.bdims, np.uint8)
    if mode == "voxel":
        vox = volume.device_voxels()
        _lib.check(L.pdm_block_any_lut(_lib.ptr(vox), volume.bits, *volume.dims, grid.b,
                                       _lib.ptr(nz), _lib.ptr(out), st), "pdm_block_any_lut")
    else:
        mins, maxs = _minmax_device(volume, grid, minmax)
        _lib.check(L.pdm_occupancy_minmax_prefix(_lib.ptr(mins), _lib.ptr(maxs), volume.bits,
                                                 grid.num_blocks, _lib.ptr(prefix),
                                                 _lib.ptr(out), st),
                   "pdm_occupancy_minmax_prefix")
    device.complete()
    return OccupancyMap(b=grid.b, bdims=grid.bdims, occupied=out)


def distance_transform(occ: OccupancyMap) -> DistanceMap:
    """Chessboard distance in blocks to the nearest occupied block, clamped at
    255 (acceleration.py:177-181; exact, bit-identical to chamfer_chebyshev)."""
    L = _lib.lib()
    src = occ.device()
    out = device.empty(occ.bdims, np.uint8)
    _lib.check(L.pdm_distance_transform(_lib.ptr(src), *occ.bdims, _lib.ptr(out),
                                        _lib.stream_handle()), "pdm_distance_transform")
    device.complete()
    return DistanceMap(b=occ.b, bdims=occ.bdims, dist=out)


def standard_distance_map(volume: Volume, grid: BlockGrid, tf: TransferFunction,
                          mode: str = "voxel", minmax=None) -> DistanceMap:
    """Full recompute for one TF: occupancy scan + distance transform
    (acceleration.py:184-196, the Deakin & Knackstedt baseline), fused: the
    occupancy kernel writes the transform's {0, 255} seed into D directly
    (pdm_standard_distance_map_voxel / _minmax), the passes run in place.

    A TF whose support is every intensity or none makes every block occupied
    (each block holds a voxel, and its apron range meets the support) or none:
    D is then all 0 / all 255 without a volume pass -- the reference's block
    scans exit at the first voxel or find nothing (_kernels.py:113-134).  The
    support size comes back from the device (4 bytes) to pick the path."""
    nz, prefix = _tf_support(volume, grid, tf, mode, prefix_too=True)
    L = _lib.lib()
    st = _lib.stream_handle()
    out = device.empty(grid.bdims, np.uint8)
    span = 1 << volume.bits
    support = int(prefix[span].item())  # waits for the support kernels only
    if support == 0 or support == span:
        _lib.check(L.pdm_fill_u8(_lib.ptr(out), out.numel(), 255 if support == 0 else 0, st),
                   "pdm_fill_u8")
    elif mode == "voxel":
        vox = volume.device_voxels()
        _lib.check(L.pdm_standard_distance_map_voxel(_lib.ptr(vox), volume.bits, *volume.dims,
                                                     grid.b, _lib.ptr(nz), _lib.ptr(out), st),
                   "pdm_standard_distance_map_voxel")
    else:
        mins, maxs = _minmax_device(volume, grid, minmax)
        _lib.check(L.pdm_standard_distance_map_minmax(_lib.ptr(mins), _lib.ptr(maxs),
                                                      volume.bits, *grid.bdims,
                                                      _lib.ptr(prefix), _lib.ptr(out), st),
                   "pdm_standard_distance_map_minmax")
    device.complete()
    return DistanceMap(b=grid.b, bdims=grid.bdims, dist=out)


def partition_mask(volume: Volume, grid: BlockGrid, scheme: PartitionScheme,
                   mode: str = "range_apron"):
    """Per-block partition bitmask [num_blocks, ceil(n/32)] uint32 on the device
    (the POM of every partition at once; acceleration.py:218-229)."""
    L = _lib.lib()
    words = _mask_words(scheme.n)
    mask = device.empty((grid.num_blocks, words), np.int32)
    vox = volume.device_voxels()
    pid = scheme.device_pid_lut()
    fn = L.pdm_partition_mask_voxel if mode == "voxel" else L.pdm_partition_mask_range_apron
    _lib.check(fn(_lib.ptr(vox), volume.bits, *volume.dims, grid.b, _lib.ptr(pid), scheme.n,
                  _lib.ptr(mask), words, _lib.stream_handle()), f"partition mask ({mode})")
    return mask


def build_pdm_set(volume: Volume, grid: BlockGrid, scheme: PartitionScheme,
                  mode: str = "range_apron") -> PdmSet:
    """Every partition's occupancy and distance map in one shot
    (acceleration.py:199-241).  init_seconds is measured to device completion."""
    _require_mode(mode)
    check_pair(volume, grid)
    if scheme.intensity_span != (1 << volume.bits):
        raise VolumeError(
            f"scheme spans {scheme.intensity_span} intensities, volume needs {1 << volume.bits}")
    L = _lib.lib()
    torch = device.torch()
    torch.cuda.synchronize()
    start = time.perf_counter()
    mask = partition_mask(volume, grid, scheme, mode)
    pitch = device.plane_pitch(grid.num_blocks)
    storage = device.empty((scheme.n, pitch), np.uint8)
    pset = PdmSet(grid=grid, scheme=scheme, occupancy_mode=mode, storage=storage)
    pset._delta_ok = grid.bdims[2] % 16 == 0
    if _packed_enabled():
        # the packed merge planes are part of the precompute; the z pass
        # writes them itself when it can (pdm_distance_transform_mask_packed)
        pending = pset._alloc_packed()
        nib, nib_pitch, base, base_pitch, bad = pending
        tb = pset._alloc_tile_bounds()
        _lib.check(L.pdm_distance_transform_mask_packed(
            _lib.ptr(mask), mask.shape[1], scheme.n, *grid.bdims, _lib.ptr(storage), pitch,
            _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, _lib.ptr(bad),
            _lib.ptr(tb) if tb is not None else None, _lib.stream_handle()),
            "pdm_distance_transform_mask_packed")
    else:
        pending, tb = False, None
        _lib.check(L.pdm_distance_transform_mask(_lib.ptr(mask), mask.shape[1], scheme.n,
                                                 *grid.bdims, _lib.ptr(storage), pitch,
                                                 _lib.stream_handle()),
                   "pdm_distance_transform_mask")
    pset._finish_pack(pending, tb)  # (+ the merge's tile bounds)
    torch.cuda.synchronize()
    pset.init_seconds = time.perf_counter() - start
    return pset


def combine(pdm_set: PdmSet, selection: PartitionSelection,
            max_maps_per_pass: int | None = None) -> DistanceMap:
    """Element-wise min of the selected partitions' maps, all-255 for an empty
    selection (acceleration.py:244-276).  One kernel pass reads each selected
    map once; max_maps_per_pass is validated like the reference and does not
    change the result (the reference guarantees chunked == direct).

    Like the reference, the call returns a finished map: the merge runs into a
    fresh HBM buffer (never aliasing a PDM) and the call waits for it.  The
    host view ``.dist`` is made on first access: for large maps D' crosses
    PCIe re-encoded in a compact form and is expanded on the host
    (pdm_dprime_to_host).  update_from_tf / combine_flags_into are the
    asynchronous, caller-buffer variants."""
    if selection.n != pdm_set.n:
        raise SelectionError(
            f"selection is over {selection.n} partitions, set holds {pdm_set.n}")
    grid = pdm_set.grid
    flags = selection.device_flags()
    if (flags is not None and selection._selected is None and max_maps_per_pass is None
            and pdm_set.n <= _MAX_FLAGS):
        # selection held on the device (select_partitions_device, the session)
        out = device.empty(grid.bdims, np.uint8)
        combine_flags_into(pdm_set, flags, out)
    else:
        sel = selection.indices0()
        if sel.size and max_maps_per_pass is not None and max_maps_per_pass < 1:
            raise ValueError(f"max_maps_per_pass must be >= 1, got {max_maps_per_pass}")
        out = device.empty(grid.bdims, np.uint8)
        if 0 < sel.size <= _MAX_PACKED_SEL and _host_reader(pdm_set):
            return _combine_with_host_view(pdm_set, sel, out)
        _combine_indices(pdm_set, sel, out)
    device.complete()
    dm = DistanceMap._of_device(grid.b, grid.bdims, out)
    if _host_packed_pays(pdm_set):
        probe = _HostReadProbe()
        pdm_set._last_probe = probe
        dm._probe = probe
        dm._host_fill = lambda host: _dprime_to_host(pdm_set, out, host)
    return dm


class _HostReadProbe:
    """Whether the host view of one combine() result was read."""

    __slots__ = ("read", "dual")

    def __init__(self, dual: bool = False):
        self.read = False
        self.dual = dual


def _host_reader(pdm_set: PdmSet) -> bool:
    """Should this combine() also stream D''s host view?  Yes while the
    caller keeps reading ``.dist`` of its results (a CLI / service / script
    that consumes D' on the host): the last result of this set had its host
    view read.  A device consumer (the ray marcher, the reference's
    measure_ms(combine)) never reads it, so it never pays for PCIe.
    PDM_HOST_SPECULATE=0 turns this off (A/B)."""
    probe = getattr(pdm_set, "_last_probe", None)
    if probe is None or not probe.read or not _SPECULATE:
        return False
    return _host_packed_pays(pdm_set) and _host_format(pdm_set) == 3


_SPECULATE = os.environ.get("PDM_HOST_SPECULATE", "1") != "0"


def _combine_with_host_view(pdm_set: PdmSet, sel: np.ndarray, out) -> DistanceMap:
    """combine() for a host reader, one pass (pdm_combine_packed_host): the
    merge writes D' into ``out`` (HBM) and its sparse delta form into pinned
    staging; the host expands each piece while the next is merged.  Returns
    with both copies complete, so ``.dist`` is free."""
    L = _lib.lib()
    grid = pdm_set.grid
    nib, nib_pitch, base, base_pitch = pdm_set.packed()
    stage, _ = pdm_set._host_stage()
    host = device.host_buffer(grid.bdims)
    nb = grid.num_blocks
    pieces = max(1, min(16, (-(-nb // 32)) // _HOST_PIECE_ITEMS))
    _lib.check(L.pdm_combine_packed_host(_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                                         pdm_set.tile_bounds_ptr(), nb, pdm_set.n, None,
                                         sel.ctypes.data, int(sel.size),
                                         _lib.ptr(out), _lib.ptr(stage), host.ctypes.data,
                                         pieces, _lib.stream_handle()),
               "pdm_combine_packed_host")
    dm = DistanceMap(b=grid.b, bdims=grid.bdims, dist=out)
    dm._host = host
    probe = _HostReadProbe(dual=True)
    pdm_set._last_probe = probe
    dm._probe = probe
    return dm


_RAW_MAX_K = None


def _raw_max_k() -> int:
    """Largest selection merged from the raw planes (pdm_combine_raw_max_k)."""
    global _RAW_MAX_K
    if _RAW_MAX_K is None:
        _RAW_MAX_K = int(_lib.lib().pdm_combine_raw_max_k())
    return _RAW_MAX_K


def _combine_indices(pdm_set: PdmSet, sel: np.ndarray, out) -> None:
    """K7 over a host index list (0-based), into ``out`` (enqueued only)."""
    L = _lib.lib()
    grid = pdm_set.grid
    # small selections: the raw planes (the packed merge is latency-bound there,
    # pdm_combine_flags_auto)
    ptrs = (pdm_set._packed_args() if _raw_max_k() < sel.size <= _MAX_PACKED_SEL else None)
    if ptrs is not None:
        _lib.check(L.pdm_combine_packed(*ptrs, grid.num_blocks, pdm_set.n, sel.ctypes.data,
                                        int(sel.size), out.data_ptr(), None,
                                        _lib.stream_handle()), "pdm_combine_packed")
        return
    storage = pdm_set.storage if sel.size else None
    _lib.check(L.pdm_combine(_lib.ptr(storage) if storage is not None else None,
                             pdm_set.plane_pitch, grid.num_blocks, max(pdm_set.n, 1),
                             sel.ctypes.data if sel.size else None, int(sel.size),
                             _lib.ptr(out), _lib.stream_handle()), "pdm_combine")


_HOST_PIECE_ITEMS = 1 << 18  # 32-block items per pipelined piece (2 pieces at config c)
_HOST_PACKED_MIN_BLOCKS = 1 << 22  # below ~4 MB of D' PCIe time is small: raw zero-copy


def _host_packed_pays(pdm_set: PdmSet) -> bool:
    """Ship D' compact to the host only when the PCIe bytes it saves matter
    (config a/b maps of 0.26-2 MB measured faster raw: no expansion pass).
    The compact forms rely on D' being a min of distance fields (packable set)."""
    return pdm_set.grid.num_blocks >= _HOST_PACKED_MIN_BLOCKS and pdm_set.packed() is not None


def _dprime_to_host(pdm_set: PdmSet, d_dev, host: np.ndarray) -> None:
    """The host view of a finished D' (pdm_dprime_to_host): D' re-encoded in a
    compact form (sparse deltas: ~1.8 MB instead of 16.8 MB at config c) is
    stored into pinned staging over PCIe in pieces, and the host expands
    piece i while piece i+1 is still in flight."""
    L = _lib.lib()
    stage, stage_base = pdm_set._host_stage()
    nb = pdm_set.grid.num_blocks
    pieces = max(1, min(16, (-(-nb // 32)) // _HOST_PIECE_ITEMS))
    _lib.check(L.pdm_dprime_to_host(_lib.ptr(d_dev), nb, _lib.ptr(stage), _lib.ptr(stage_base),
                                    host.ctypes.data, pieces, _host_format(pdm_set),
                                    _lib.stream_handle()), "pdm_dprime_to_host")


def _host_format(pdm_set: PdmSet) -> int:
    """Form of D' on the PCIe link (pdm_merge_packed_to_host `format`): 3 =
    sparse deltas (default), 2 = deltas, 1 = nibbles.  The delta forms need
    chunks that never straddle a z row (bz % 16 == 0).  PDM_HOST_FORMAT
    picks a lower one for A/B measurements."""
    want = int(os.environ.get("PDM_HOST_FORMAT", "3"))
    if want not in (1, 2, 3):
        raise ValueError(f"PDM_HOST_FORMAT must be 1, 2 or 3, got {want}")
    return want if pdm_set._delta_ok else 1


def update_from_tf(pdm_set: PdmSet, tf, out=None, flags=None) -> DistanceMap:
    """Fused device-side TF-change update: selection (K8) + merge (K7) with the
    selection kept in HBM -- two kernels, no host round trip.  ``tf`` is a
    TransferFunction or a device-resident f64 alpha tensor of length 2^bits.
    Equivalent to combine(pdm_set, select_partitions(tf, scheme))."""
    alpha = alpha_to_device(tf) if isinstance(tf, TransferFunction) else tf
    flags = select_partitions_device(alpha, pdm_set.scheme, flags)
    return combine_flags_into(pdm_set, flags, out)


def combine_flags_into(pdm_set: PdmSet, flags, out=None, count_zeros: bool = False) -> DistanceMap:
    """K7 with a device-resident selection (uint8 flags[n], e.g. from
    select_partitions_device) writing into ``out`` (allocated if None).
    count_zeros: the packed merge also counts D''s zero blocks, so the result's
    occupied_fraction needs no second pass (the live session's report)."""
    L = _lib.lib()
    grid = pdm_set.grid
    if out is None:
        out = device.empty(grid.bdims, np.uint8)
    packed = pdm_set.packed() if out.is_cuda else None  # host out: see combine()
    if packed is not None:
        nib, nib_pitch, base, base_pitch = packed
        zeros = device.empty((1,), np.int64) if count_zeros else None
        # raw planes beside the packed ones: small selections merge those
        _lib.check(L.pdm_combine_flags_auto(_lib.ptr(pdm_set.storage), pdm_set.plane_pitch,
                                            _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                                            pdm_set.tile_bounds_ptr(), grid.num_blocks,
                                            pdm_set.n, _lib.ptr(flags), _lib.ptr(out),
                                            _lib.ptr(zeros) if zeros is not None else None,
                                            _lib.stream_handle()),
                   "pdm_combine_flags_auto")
        dm = DistanceMap(b=grid.b, bdims=grid.bdims, dist=out)
        dm._zero_count = zeros
        return dm
    _lib.check(L.pdm_combine_flags(_lib.ptr(pdm_set.storage), pdm_set.plane_pitch,
                                   grid.num_blocks, pdm_set.n, _lib.ptr(flags), _lib.ptr(out),
                                   _lib.stream_handle()), "pdm_combine_flags")
    return DistanceMap(b=grid.b, bdims=grid.bdims, dist=out)


# --- persistence (acceleration.py:279-354 formats) -----------------------------

def save_distance_map(dm: DistanceMap, path) -> None:
    """'PDMD' + <4I (b, bx, by, bz) + raw uint8 payload."""
    Path(path).write_bytes(_MAP_MAGIC + struct.pack("<4I", dm.b, *dm.bdims) + dm.dist.tobytes())


def load_distance_map(path) -> DistanceMap:
    raw = Path(path).read_bytes()
    if raw[:4] != _MAP_MAGIC:
        raise VolumeError(f"{path} is not a distance map dump")
    b, bx, by, bz = struct.unpack_from("<4I", raw, 4)
    payload = np.frombuffer(raw, dtype=np.uint8, offset=20)
    if payload.size != bx * by * bz:
        raise VolumeError(f"{path} payload size does not match header dims")
    return DistanceMap(b=b, bdims=(bx, by, bz), dist=payload.reshape((bx, by, bz)).copy())


_IO_CHUNK = 32 << 20  # bytes per pinned staging buffer (two in flight)


def _stage_buffers():
    t = device.torch()
    return ([t.empty(_IO_CHUNK, dtype=t.uint8, pin_memory=True) for _ in range(2)],
            [t.cuda.Event() for _ in range(2)])


def _set_header(pdm_set: PdmSet) -> bytes:
    g = pdm_set.grid
    head = _SET_MAGIC + struct.pack("<9I", g.b, *g.dims, *g.bdims, pdm_set.n,
                                    0 if pdm_set.occupancy_mode == "voxel" else 1)
    return head + b"".join(struct.pack("<2I", lo, hi) for lo, hi in pdm_set.scheme.bounds())


def save_pdm_set(pdm_set: PdmSet, path) -> None:
    """'PDMS' + <9I (b, dims, bdims, n, mode) + n x <2I bounds + n raw maps
    (acceleration.py:297-315 byte format).  Device-resident planes stream to
    the file through two pinned buffers (the D2H of chunk i+1 overlaps the
    write of chunk i); a set of host maps is written as is (no device)."""
    nb = pdm_set.grid.num_blocks
    with open(path, "wb") as f:
        f.write(_set_header(pdm_set))
        if pdm_set._storage is None:
            for dm in pdm_set.pdms:
                f.write(np.ascontiguousarray(dm.dist, dtype=np.uint8).tobytes())
            return
        st = pdm_set.storage
        bufs, evs = _stage_buffers()
        jobs = [(p, o, min(_IO_CHUNK, nb - o)) for p in range(pdm_set.n)
                for o in range(0, nb, _IO_CHUNK)]
        pending = None
        for i, (p, o, ln) in enumerate(jobs):
            k = i % 2
            bufs[k][:ln].copy_(st[p, o:o + ln], non_blocking=True)
            evs[k].record()
            if pending is not None:
                evs[pending[0]].synchronize()
                f.write(memoryview(bufs[pending[0]][:pending[1]].numpy()))
            pending = (k, ln)
        if pending is not None:
            evs[pending[0]].synchronize()
            f.write(memoryview(bufs[pending[0]][:pending[1]].numpy()))


def _read_set_header(f, path):
    """(grid, scheme, mode, payload offset) of a 'PDMS' dump, validated like
    the reference's load_pdm_set (acceleration.py:318-354)."""
    raw = f.read(40)
    if raw[:4] != _SET_MAGIC or len(raw) < 40:
        raise VolumeError(f"{path} is not a partition set dump")
    vals = struct.unpack_from("<9I", raw, 4)
    b, dims, bdims, n = vals[0], vals[1:4], tuple(vals[4:7]), vals[7]
    mode = "voxel" if vals[8] == 0 else "range_apron"
    grid = BlockGrid.for_dims(dims, b)
    if grid.bdims != bdims:
        raise VolumeError(f"{path} header block dims are inconsistent")
    braw = f.read(8 * n)
    if len(braw) != 8 * n:
        raise VolumeError(f"{path} payload size does not match header")
    bounds = [struct.unpack_from("<2I", braw, 8 * i) for i in range(n)]
    off = 40 + 8 * n
    if os.fstat(f.fileno()).st_size - off != n * grid.num_blocks:
        raise VolumeError(f"{path} payload size does not match header")
    scheme = PartitionScheme(tuple(Partition(lo, hi) for lo, hi in bounds))
    return grid, scheme, mode, off


def _read_pdm_set_host(path):
    """Host-side parse of a 'PDMS' dump: (grid, scheme, mode, maps uint8
    [n, num_blocks] memory-mapped) -- no device."""
    with open(path, "rb") as f:
        grid, scheme, mode, off = _read_set_header(f, path)
    maps = np.memmap(path, dtype=np.uint8, mode="r", offset=off,
                     shape=(scheme.n, grid.num_blocks))
    return grid, scheme, mode, maps


def load_pdm_set(path) -> PdmSet:
    """Reads a 'PDMS' dump straight into one [n][plane_pitch] device
    allocation: the payload streams through two pinned buffers (the read of
    chunk i+1 overlaps the DMA of chunk i), then the merge's packed planes are
    built on the device.  The PCIe delta forms of D' are enabled only if every
    chunk of every loaded map is 1-Lipschitz (pdm_count_nonlipschitz_chunks)."""
    with open(path, "rb") as f:
        grid, scheme, mode, off = _read_set_header(f, path)
        n, nb = scheme.n, grid.num_blocks
        storage = device.empty((n, device.plane_pitch(nb)), np.uint8)
        bufs, evs = _stage_buffers()
        used = [False, False]
        i = 0
        for p in range(n):
            for o in range(0, nb, _IO_CHUNK):
                ln = min(_IO_CHUNK, nb - o)
                k = i % 2
                if used[k]:
                    evs[k].synchronize()  # the DMA out of this buffer has finished
                view = bufs[k][:ln].numpy()
                if f.readinto(memoryview(view)) != ln:
                    raise VolumeError(f"{path} payload size does not match header")
                storage[p, o:o + ln].copy_(bufs[k][:ln], non_blocking=True)
                evs[k].record()
                used[k] = True
                i += 1
    pset = PdmSet(grid=grid, scheme=scheme, occupancy_mode=mode, init_seconds=0.0,
                  storage=storage)
    L = _lib.lib()
    bad = device.empty((1,), np.int32)
    _lib.check(L.pdm_count_nonlipschitz_chunks(_lib.ptr(storage), pset.plane_pitch, nb, n,
                                               _lib.ptr(bad), _lib.stream_handle()),
               "pdm_count_nonlipschitz_chunks")
    pset.packed()  # pack at load, not in the first merge
    pset._delta_ok = int(bad.item()) == 0
    device.complete()
    return pset
