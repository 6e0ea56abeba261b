"""Multi-GPU x-slab sharding of the PDM precompute.

The volume is split into contiguous slabs of whole block planes along x, the
slowest memory axis ([x][y][z] C-order, z contiguous) -- the north_star's
"z-slabs" in memory terms.  One process per GPU; each rank holds its volume
slab, its slab of every partition map and (after an update) its slab of D'.

* TF-change update (select + merge): embarrassingly parallel, no collective.
* POM build, voxel mode: local.  range_apron mode: a block's apron reaches one
  voxel plane into each neighbour slab, so neighbours swap one boundary voxel
  plane (send/recv over NCCL) and fold its apron min/max into their first/last
  block plane (pdm_minmax_fold).
* Distance transform: pass x runs along the shard axis, locally, then each
  rank contributes its two edge planes per partition (the distance from its
  first/last block plane to its nearest occupied block) to one all_gather of
  2 * n * by * bz bytes per rank; pdm_dt_slab_fold folds every other slab's
  nearest occupied block into the local 1-D distances, after which passes y
  and z are local.  Bit-exact against the single-GPU transform (min over
  slabs of clamped distances composes exactly).

Collectives go through torch.distributed (NCCL on GPUs; gloo in the CPU
tests and the 2-process single-GPU test, with CUDA tensors staged via host).
The per-slab compute is an ``ops`` object: ``GpuOps`` (libpdm_b200 kernels)
in the product; tests substitute a host implementation to exercise the
collective logic on CPU with gloo.
"""

from __future__ import annotations

import numpy as np

from . import _lib, device
from .acceleration import PdmSet, _require_mode
from .transfer import PartitionScheme
from .volume import BlockGrid, Volume, VolumeError


class GpuOps:
    """Per-slab compute on CUDA tensors via libpdm_b200."""

    def empty(self, shape, np_dtype):
        return device.empty(shape, np_dtype)

    def voxels(self, volume):
        return volume.device_voxels()

    def plane(self, vol_t, x):
        return vol_t[x: x + 1].contiguous()

    def block_min_max(self, vol_t, bits, b):
        L = _lib.lib()
        dims = tuple(vol_t.shape)
        bd = tuple(-(-d // b) for d in dims)
        dt = np.uint8 if bits == 8 else np.uint16
        mins, maxs = self.empty(bd, dt), self.empty(bd, dt)
        _lib.check(L.pdm_block_min_max(_lib.ptr(vol_t), bits, *dims, b, _lib.ptr(mins),
                                       _lib.ptr(maxs), _lib.stream_handle()), "pdm_block_min_max")
        return mins, maxs

    def fold_minmax(self, mins_plane, maxs_plane, pmins, pmaxs, bits):
        L = _lib.lib()
        _lib.check(L.pdm_minmax_fold(_lib.ptr(mins_plane), _lib.ptr(maxs_plane), _lib.ptr(pmins),
                                     _lib.ptr(pmaxs), bits, mins_plane.numel(),
                                     _lib.stream_handle()), "pdm_minmax_fold")

    def mask_from_minmax(self, mins, maxs, bits, scheme):
        L = _lib.lib()
        words = (scheme.n + 31) // 32
        mask = self.empty((mins.numel(), words), np.int32)
        _lib.check(L.pdm_partition_mask_minmax(_lib.ptr(mins), _lib.ptr(maxs), bits, mins.numel(),
                                               _lib.ptr(scheme.device_pid_lut()), scheme.n,
                                               _lib.ptr(mask), words, _lib.stream_handle()),
                   "pdm_partition_mask_minmax")
        return mask

    def mask_voxel(self, vol_t, bits, b, scheme):
        L = _lib.lib()
        dims = tuple(vol_t.shape)
        nb = int(np.prod([-(-d // b) for d in dims]))
        words = (scheme.n + 31) // 32
        mask = self.empty((nb, words), np.int32)
        _lib.check(L.pdm_partition_mask_voxel(_lib.ptr(vol_t), bits, *dims, b,
                                              _lib.ptr(scheme.device_pid_lut()), scheme.n,
                                              _lib.ptr(mask), words, _lib.stream_handle()),
                   "pdm_partition_mask_voxel")
        return mask

    def pass_x(self, mask, n, bdims, storage, pitch):
        L = _lib.lib()
        _lib.check(L.pdm_dt_pass_x_mask(_lib.ptr(mask), mask.shape[1], n, *bdims,
                                        _lib.ptr(storage), pitch, _lib.stream_handle()),
                   "pdm_dt_pass_x_mask")

    def edges(self, storage, pitch, n, bdims):
        L = _lib.lib()
        e = self.empty((2, n, bdims[1], bdims[2]), np.uint8)
        _lib.check(L.pdm_dt_slab_edges(_lib.ptr(storage), pitch, n, *bdims, _lib.ptr(e),
                                       _lib.stream_handle()), "pdm_dt_slab_edges")
        return e

    def fold(self, storage, pitch, n, bdims, edges_all, world, rank, slab_x0):
        L = _lib.lib()
        x0 = np.ascontiguousarray(slab_x0, dtype=np.int64)
        _lib.check(L.pdm_dt_slab_fold(_lib.ptr(storage), pitch, n, *bdims, _lib.ptr(edges_all),
                                      world, rank, x0.ctypes.data, _lib.stream_handle()),
                   "pdm_dt_slab_fold")

    def pass_yz(self, storage, pitch, n, bdims):
        L = _lib.lib()
        _lib.check(L.pdm_dt_pass_yz(_lib.ptr(storage), pitch, n, *bdims, _lib.stream_handle()),
                   "pdm_dt_pass_yz")


def slab_bounds(nx: int, b: int, world: int) -> list[int]:
    """Voxel x0 of each slab (+ nx): whole block planes, as even as possible."""
    bx = -(-nx // b)
    per, rem = divmod(bx, world)
    starts, acc = [], 0
    for r in range(world):
        starts.append(min(acc * b, nx))
        acc += per + (r < rem)
    return starts + [nx]


class _Comm:
    """torch.distributed collectives for the sharded build.  NCCL moves CUDA
    tensors directly (NVLink); other backends (gloo: CPU tests, and the
    2-process single-GPU test) stage CUDA tensors through host memory."""

    def __init__(self, group):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def _out(self, t):
        return t if self.nccl or not t.is_cuda else t.cpu()

    def all_gather(self, t):
        """[world, *t.shape] of every rank's t, on t's device."""
        import torch

        src = self._out(t).contiguous()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        return torch.stack(parts).to(t.device)

    def exchange(self, sends, recvs):
        """Point-to-point: sends = [(tensor, peer)], recvs = [(like_tensor,
        peer)]; returns the received tensors (on the like tensors' devices)."""
        P2P = self.dist.P2POp
        ops, bufs = [], []
        for t, peer in sends:
            ops.append(P2P(self.dist.isend, self._out(t).contiguous(), peer, self.group))
        for like, peer in recvs:
            buf = self._out(like)
            bufs.append((buf, like))
            ops.append(P2P(self.dist.irecv, buf, peer, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return [buf.to(like.device) if buf is not like else buf for buf, like in bufs]


def _exchange_planes(vol_t, ops, comm: _Comm):
    """Swap boundary voxel planes with the x-neighbours.  Returns (below, above):
    the neighbour's plane at x0-1 and x1 (None at the volume ends)."""
    rank, world = comm.rank, comm.world
    nxl = vol_t.shape[0]
    shape = (1,) + tuple(vol_t.shape[1:])
    sends, recvs = [], []
    if rank > 0:
        sends.append((ops.plane(vol_t, 0), rank - 1))
        recvs.append((ops.empty(shape, _np_dtype(vol_t)), rank - 1))
    if rank < world - 1:
        sends.append((ops.plane(vol_t, nxl - 1), rank + 1))
        recvs.append((ops.empty(shape, _np_dtype(vol_t)), rank + 1))
    got = comm.exchange(sends, recvs)
    below = got.pop(0) if rank > 0 else None
    above = got.pop(0) if rank < world - 1 else None
    return below, above


def _np_dtype(t):
    return np.uint8 if t.element_size() == 1 else np.uint16


def build_pdm_set_sharded(volume: Volume, b: int, scheme: PartitionScheme,
                          mode: str = "range_apron", bx0: int | None = None, group=None,
                          ops=None) -> PdmSet:
    """build_pdm_set over an x-slab of a volume split across the ranks of
    ``group``.  ``volume`` is this rank's slab (its x0 must be a multiple of b
    and every slab but the last must hold whole blocks); the result is this
    rank's slab of every partition's distance map, bit-identical to the
    corresponding planes of the single-device build_pdm_set.

    Validation is agreed across ranks before any data moves: the slab table
    all_gather carries each rank's error flag, so a bad slab makes EVERY rank
    raise VolumeError instead of leaving its peers waiting in a collective."""
    import torch

    _require_mode(mode)
    if scheme.intensity_span != (1 << volume.bits):
        raise VolumeError(
            f"scheme spans {scheme.intensity_span} intensities, volume needs {1 << volume.bits}")
    ops = ops or GpuOps()
    comm = _Comm(group)
    world, rank = comm.world, comm.rank
    vol_t = ops.voxels(volume)
    grid = BlockGrid.for_dims(volume.dims, b)
    bdims, n = grid.bdims, scheme.n

    # slab table in block planes (every rank learns every slab's start) + error flags
    partial = int(volume.dims[0] % b != 0)  # legal on the last rank only
    mine = torch.tensor([-1 if bx0 is None else bx0, bdims[0], partial], dtype=torch.int64)
    if comm.nccl:
        mine = mine.cuda()
    table = comm.all_gather(mine).cpu().numpy()
    sizes = table[:, 1]
    starts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    for r in range(world):
        if table[r, 2] and r < world - 1:
            raise VolumeError(f"rank {r}: only the last slab may end inside a block")
        if table[r, 0] >= 0 and table[r, 0] != starts[r]:
            raise VolumeError(f"rank {r}: slab starts at block {table[r, 0]}, "
                              f"expected {starts[r]}")

    below = above = None
    if mode == "range_apron":
        below, above = _exchange_planes(vol_t, ops, comm)
    storage, pitch, edges = slab_phase_local(vol_t, volume.bits, b, scheme, mode, below, above,
                                             ops)
    edges_all = comm.all_gather(edges).contiguous()
    slab_phase_fold(storage, pitch, n, bdims, edges_all, world, rank, starts, ops)
    pset = PdmSet(grid=grid, scheme=scheme, occupancy_mode=mode, storage=storage)
    pset.slab = (int(starts[rank]), int(starts[rank + 1]), int(starts[-1]))
    pset._delta_ok = bdims[2] % 16 == 0  # distance-transform output (see build_pdm_set)
    if storage.is_cuda:
        pset.packed()  # pack the final planes now, not in the first merge
    return pset


def torch_nccl_comm(group=None) -> int:
    """The ncclComm_t (as an int) of a torch.distributed NCCL process group
    (ProcessGroupNCCL._comm_ptr), forcing its lazy creation first."""
    import torch
    import torch.distributed as dist

    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    backend = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    ptr = int(backend._comm_ptr())
    if ptr == 0:  # communicator not created yet: one tiny collective does it
        dist.all_reduce(torch.zeros(1, device="cuda"), group=group)
        ptr = int(backend._comm_ptr())
    return ptr


def build_pdm_set_sharded_nccl(volume: Volume, b: int, scheme: PartitionScheme,
                               mode: str = "range_apron", bx0: int | None = None,
                               comm: int | None = None, group=None) -> PdmSet:
    """build_pdm_set_sharded as ONE library call over an NCCL communicator
    (pdm_build_pdm_set_slab_nccl, the C-ABI multi-GPU entry of SURVEY.md §8b
    item 5): slab table, boundary planes, edge all_gather, fold, y/z passes
    and the packed planes all enqueued on the current stream.  ``comm`` is an
    ncclComm_t (default: the NCCL communicator of ``group`` / the default
    torch.distributed group)."""
    _require_mode(mode)
    if scheme.intensity_span != (1 << volume.bits):
        raise VolumeError(
            f"scheme spans {scheme.intensity_span} intensities, volume needs {1 << volume.bits}")
    L = _lib.lib()
    if comm is None:
        comm = torch_nccl_comm(group)
    vol_t = volume.device_voxels()
    grid = BlockGrid.for_dims(volume.dims, b)
    n = scheme.n
    pitch = device.plane_pitch(grid.num_blocks)
    storage = device.empty((n, pitch), np.uint8)
    pset = PdmSet(grid=grid, scheme=scheme, occupancy_mode=mode, storage=storage)
    import ctypes

    ws_bytes = int(L.pdm_build_pdm_set_slab_nccl_workspace(
        _comm_size(L, comm), volume.bits, *volume.dims, b, n))
    if ws_bytes < 0:
        raise ValueError("pdm_build_pdm_set_slab_nccl_workspace: bad sizes")
    ws = device.empty((ws_bytes,), np.uint8)
    packed = pset._alloc_packed() if n else False
    nib, nib_pitch, base, base_pitch, bad = packed
    slab = (ctypes.c_int64 * 3)()
    _lib.check(L.pdm_build_pdm_set_slab_nccl(
        comm, _lib.ptr(vol_t), volume.bits, *volume.dims, b, _lib.ptr(scheme.device_pid_lut()),
        n, 0 if mode == "voxel" else 1, -1 if bx0 is None else int(bx0), _lib.ptr(storage),
        pitch, _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, _lib.ptr(bad),
        _lib.ptr(ws), ws_bytes, ctypes.addressof(slab), _lib.stream_handle()),
        "pdm_build_pdm_set_slab_nccl")
    pset._finish_pack(packed)
    pset.slab = (int(slab[0]), int(slab[1]), int(slab[2]))
    pset._delta_ok = grid.bdims[2] % 16 == 0
    device.complete()
    return pset


def _comm_size(L, comm) -> int:
    """Ranks of an ncclComm_t (for the workspace size)."""
    world = int(L.pdm_nccl_comm_count(comm))
    if world < 1:
        raise RuntimeError("pdm_nccl_comm_count: not a valid NCCL communicator")
    return world


def slab_phase_local(vol_t, bits: int, b: int, scheme: PartitionScheme, mode: str, below, above,
                     ops):
    """Everything a rank does before the exchange: its POM (folding in the
    neighbours' boundary voxel planes ``below``/``above`` in range_apron mode),
    the local 1-D distance along x, and its edge planes.  Returns
    (storage [n, pitch], pitch, edges [2, n, by, bz])."""
    dims = tuple(vol_t.shape)
    bdims = tuple(-(-d // b) for d in dims)
    n = scheme.n
    if mode == "voxel":
        mask = ops.mask_voxel(vol_t, bits, b, scheme)
    else:
        mins, maxs = ops.block_min_max(vol_t, bits, b)
        if below is not None:
            pm, px = ops.block_min_max(below, bits, b)
            ops.fold_minmax(mins[0:1], maxs[0:1], pm, px, bits)
        if above is not None:
            pm, px = ops.block_min_max(above, bits, b)
            ops.fold_minmax(mins[-1:], maxs[-1:], pm, px, bits)
        mask = ops.mask_from_minmax(mins, maxs, bits, scheme)
    nb = bdims[0] * bdims[1] * bdims[2]
    pitch = device.plane_pitch(nb)
    storage = ops.empty((n, pitch), np.uint8)
    ops.pass_x(mask, n, bdims, storage, pitch)
    return storage, pitch, ops.edges(storage, pitch, n, bdims)


def slab_phase_fold(storage, pitch: int, n: int, bdims, edges_all, world: int, rank: int,
                    slab_x0, ops) -> None:
    """After the exchange: fold the other slabs' nearest occupied blocks into
    the local 1-D distances, then the local y and z passes."""
    ops.fold(storage, pitch, n, bdims, edges_all, world, rank, slab_x0)
    ops.pass_yz(storage, pitch, n, bdims)
