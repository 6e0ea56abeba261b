"""Multi-rank x-slab sharding of the PDM precompute (paper_2407_21552_b200.sharded).

* CPU: world_size 2 and 3 over gloo, per-slab compute by the host ops
  (tests/sharded_host_ops.py), every rank's slab of every PDM compared with
  the oracle's single-volume build_pdm_set -- exercises the slab table, the
  boundary-plane send/recv (range_apron) and the edge all_gather + fold.
* GPU: the same decomposition emulated on one device with the CUDA slab
  kernels (slab_phase_local on each slab, stacked edges, slab_phase_fold):
  bit-identical to the single-GPU build.  No kernel waits on another.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2407_21552_b200 as pdm
from conftest import random_structured_volume
from paper_2407_21552_b200 import sharded

CASES = [
    # dims, bits, b, n, block planes per slab (None = even split)
    ((24, 10, 12), 8, 4, 8, None),
    ((22, 9, 14), 16, 2, 5, None),   # last slab ends inside a block (22 / 2 = 11 planes)
    ((30, 7, 9), 8, 3, 40, None),    # n > 32: two mask words
    ((40, 6, 5), 8, 1, 4, [3, 30, 7]),
]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slab_planes(bx, world, planes):
    if planes is not None:
        return planes
    per, rem = divmod(bx, world)
    return [per + (r < rem) for r in range(world)]


def _worker(rank, world, port, case, mode, seed):
    from sharded_host_ops import HostOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, bits, b, n, planes = case
        rng = np.random.default_rng(seed)
        vox = random_structured_volume(rng, dims, bits)
        scheme = pdm.scheme_uniform(n, bits)
        bx = -(-dims[0] // b)
        planes = _slab_planes(bx, world, planes)[:world]
        starts = np.concatenate([[0], np.cumsum(planes)])
        x0, x1 = int(starts[rank]) * b, min(int(starts[rank + 1]) * b, dims[0])
        slab = pdm.Volume.from_array(vox[x0:x1])
        pset = sharded.build_pdm_set_sharded(slab, b, scheme, mode, bx0=int(starts[rank]),
                                             ops=HostOps())
        nb = pset.grid.num_blocks
        got = pset.storage[:, :nb].numpy().reshape((n,) + pset.grid.bdims)
        want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)[:, starts[rank]:starts[rank + 1]]
        assert pset.slab == (int(starts[rank]), int(starts[rank + 1]), bx)
        assert np.array_equal(got, want), f"rank {rank} slab mismatch ({mode})"
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_build_gloo(case, mode, world):
    if case[4] is not None and len(case[4]) != world:
        pytest.skip("explicit slab layout is for world=3")
    mp.spawn(_worker, args=(world, _free_port(), case, mode, 1234 + world), nprocs=world,
             join=True)


def test_fold_restatement_matches_full_transform():
    """The numpy fold (mirror of slab_fold_kernel) composes to the full DT."""
    from sharded_host_ops import HostOps, cone_axis, dist1d_axis0

    rng = np.random.default_rng(5)
    occ = rng.random((4, 37, 6, 5)) < 0.01
    occ[0, 2, 3, 1] = True
    full = np.stack([oracle.distance_transform(o) for o in occ])
    starts = np.array([0, 5, 6, 20, 37])
    slabs = [dist1d_axis0(occ[:, a:c].transpose(1, 0, 2, 3)).transpose(1, 0, 2, 3)
             for a, c in zip(starts[:-1], starts[1:])]
    edges = torch.from_numpy(np.stack([np.stack([s[:, 0], s[:, -1]]) for s in slabs])
                             .astype(np.uint8))
    ops = HostOps()
    for r, (a, c) in enumerate(zip(starts[:-1], starts[1:])):
        bd = (c - a, 6, 5)
        nb = int(np.prod(bd))
        st = torch.from_numpy(np.ascontiguousarray(slabs[r].reshape(4, nb).astype(np.uint8)))
        ops.fold(st, nb, 4, bd, edges, len(slabs), r, starts)
        g = st.numpy().reshape((4,) + bd)
        g = cone_axis(cone_axis(g, 2), 3)
        assert np.array_equal(g, full[:, a:c]), r


@pytest.mark.gpu
def test_sharded_build_nccl_world1(monkeypatch):
    """The NCCL plumbing of build_pdm_set_sharded (slab table and edge
    all_gathers on CUDA tensors) on a one-rank process group."""
    monkeypatch.setenv("PDM_PACKED", "1")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(77)
        dims, b, n = (32, 24, 48), 4, 12
        vox = random_structured_volume(rng, dims, 16)
        vol = pdm.Volume.from_array(vox)
        scheme = pdm.scheme_uniform(n, 16)
        for mode in ("voxel", "range_apron"):
            got = sharded.build_pdm_set_sharded(vol, b, scheme, mode, bx0=0)
            want = pdm.build_pdm_set(vol, pdm.BlockGrid.for_dims(dims, b), scheme, mode)
            assert got.slab == (0, 8, 8)
            assert np.array_equal(np.stack([d.dist for d in got.pdms]),
                                  np.stack([d.dist for d in want.pdms])), mode
            # the slab's set is packed at build time and merges like the full set
            assert got.packed() is not None
            sel = pdm.PartitionSelection(selected=frozenset({1, 4, 9, 12}), n=n)
            assert np.array_equal(pdm.combine(got, sel).dist, pdm.combine(want, sel).dist)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
@pytest.mark.parametrize("dims,bits,b,n,planes", [
    ((64, 40, 64), 16, 4, 32, [5, 1, 7, 3]),
    ((48, 20, 48), 8, 2, 12, [10, 14]),
    ((33, 16, 32), 16, 4, 40, [2, 3, 4]),  # last slab partial, two mask words
])
def test_sharded_emulated_on_one_gpu(mode, dims, bits, b, n, planes):
    rng = np.random.default_rng(sum(dims) + n)
    vox = random_structured_volume(rng, dims, bits)
    scheme = pdm.scheme_uniform(n, bits)
    full = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, b), scheme,
                             mode)
    want = np.stack([d.dist for d in full.pdms])
    ops = sharded.GpuOps()
    starts = np.concatenate([[0], np.cumsum(planes)]).astype(np.int64)
    assert starts[-1] == -(-dims[0] // b)
    world = len(planes)
    vols, outs = [], []
    for r in range(world):
        x0, x1 = int(starts[r]) * b, min(int(starts[r + 1]) * b, dims[0])
        vt = pdm.Volume.from_array(vox[x0:x1]).device_voxels()
        below = vt.new_tensor(vox[x0 - 1:x0].view(np.int16) if bits == 16 else vox[x0 - 1:x0]) \
            if (mode == "range_apron" and r > 0) else None
        above = vt.new_tensor(vox[x1:x1 + 1].view(np.int16) if bits == 16 else vox[x1:x1 + 1]) \
            if (mode == "range_apron" and r < world - 1) else None
        outs.append(sharded.slab_phase_local(vt, bits, b, scheme, mode, below, above, ops))
        vols.append(vt)
    edges_all = torch.stack([e for _, _, e in outs]).contiguous()
    for r, (storage, pitch, _) in enumerate(outs):
        bd = (int(starts[r + 1] - starts[r]),) + full.grid.bdims[1:]
        sharded.slab_phase_fold(storage, pitch, n, bd, edges_all, world, r, starts, ops)
        nb = int(np.prod(bd))
        got = storage[:, :nb].cpu().numpy().reshape((n,) + bd)
        assert np.array_equal(got, want[:, starts[r]:starts[r + 1]]), r


def _bad_slab_worker(rank, world, port, mode, q):
    """Rank 0's slab ends inside a block (illegal except on the last rank):
    every rank must raise VolumeError, none may hang in a collective."""
    from sharded_host_ops import HostOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        vox = random_structured_volume(rng, (18, 6, 8), 8)
        x0, x1 = (0, 9) if rank == 0 else (9, 18)  # b=4: 9 is inside a block
        slab = pdm.Volume.from_array(vox[x0:x1])
        try:
            sharded.build_pdm_set_sharded(slab, 4, pdm.scheme_uniform(4, 8), mode, ops=HostOps())
            q.put((rank, "no error"))
        except pdm.VolumeError as exc:
            q.put((rank, f"VolumeError: {exc}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_sharded_bad_slab_raises_on_every_rank(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bad_slab_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, "a rank hung or crashed"
    got = dict(q.get(timeout=5) for _ in range(2))
    assert all(v.startswith("VolumeError: rank 0: only the last slab") for v in got.values()), got


def _gpu_gloo_worker(rank, world, port, mode, q):
    """One rank of a 2-process sharded build on the SAME GPU: real GpuOps
    kernels per slab, collectives over gloo with the CUDA tensors staged
    through host memory (no kernel waits on another rank's kernel)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(91)
        dims, bits, b, n = (40, 24, 32), 16, 4, 12
        vox = random_structured_volume(rng, dims, bits)
        scheme = pdm.scheme_uniform(n, bits)
        xs = sharded.slab_bounds(dims[0], b, world)
        slab = pdm.Volume.from_array(vox[xs[rank]:xs[rank + 1]])
        pset = sharded.build_pdm_set_sharded(slab, b, scheme, mode, bx0=xs[rank] // b)
        assert isinstance(pset.storage, torch.Tensor) and pset.storage.is_cuda
        nb = pset.grid.num_blocks
        got = pset.storage[:, :nb].cpu().numpy().reshape((n,) + pset.grid.bdims)
        want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)[:, pset.slab[0]:pset.slab[1]]
        ok = np.array_equal(got, want)
        sel = pdm.PartitionSelection(selected=frozenset({2, 5, 11}), n=n)
        ok = ok and np.array_equal(pdm.combine(pset, sel).dist, oracle.combine(want, [2, 5, 11]))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_sharded_two_processes_one_gpu_gloo(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_gloo_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = dict(q.get(timeout=5) for _ in range(2))
    assert got == {0: True, 1: True}, got


@pytest.mark.gpu
def test_native_nccl_slab_build_world1(monkeypatch):
    """pdm_build_pdm_set_slab_nccl (the C-ABI multi-GPU entry) on a one-rank
    NCCL communicator -- torch's (ProcessGroupNCCL._comm_ptr) and one made by
    the library itself (pdm_nccl_unique_id + pdm_nccl_comm_init): PDMs,
    packed planes and merges equal the single-device build, both modes;
    a wrong expected slab start fails cleanly."""
    import ctypes

    from paper_2407_21552_b200 import _lib

    monkeypatch.setenv("PDM_PACKED", "1")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    L = _lib.lib()
    assert L.pdm_nccl_available() == 1
    uid = (ctypes.c_uint8 * 128)()
    assert L.pdm_nccl_unique_id(uid) == 0
    own = ctypes.c_void_p()
    _lib.check(L.pdm_nccl_comm_init(ctypes.byref(own), 1, uid, 0), "comm init")
    try:
        rng = np.random.default_rng(78)
        dims, b, n = (36, 24, 64), 4, 12
        vox = random_structured_volume(rng, dims, 16)
        vol = pdm.Volume.from_array(vox)
        scheme = pdm.scheme_uniform(n, 16)
        for mode in ("voxel", "range_apron"):
            want = pdm.build_pdm_set(vol, pdm.BlockGrid.for_dims(dims, b), scheme, mode)
            for comm in (None, own.value):
                got = sharded.build_pdm_set_sharded_nccl(vol, b, scheme, mode, bx0=0, comm=comm)
                assert got.slab == (0, 9, 9)
                assert np.array_equal(np.stack([d.dist for d in got.pdms]),
                                      np.stack([d.dist for d in want.pdms])), mode
                assert got.packed() is not None and got._delta_ok
                chunks = int(L.pdm_packed_chunks(got.grid.num_blocks))
                (gn, _, gb, _), (wn, _, wb, _) = got.packed(), want.packed()
                assert torch.equal(gn[:, :chunks * 8], wn[:, :chunks * 8])
                assert torch.equal(gb[:, :chunks], wb[:, :chunks])
                sel = pdm.PartitionSelection(selected=frozenset({1, 4, 9, 12}), n=n)
                assert np.array_equal(pdm.combine(got, sel).dist, pdm.combine(want, sel).dist)
        with pytest.raises(ValueError, match="expected 0"):
            sharded.build_pdm_set_sharded_nccl(vol, b, scheme, "voxel", bx0=3, comm=own.value)
    finally:
        L.pdm_nccl_comm_destroy(own)
        dist.destroy_process_group()
