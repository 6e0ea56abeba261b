"""Host (CPU) implementation of paper_2407_21552_b200.sharded's per-slab ops --
TEST INFRASTRUCTURE.  It lets the multi-rank logic of build_pdm_set_sharded
(slab table all_gather, boundary-plane send/recv, edge all_gather, fold) run
under gloo on CPU.  Block reductions come from the C oracle; the DT pieces are
numpy restatements of the CUDA kernels in csrc/dt.cu (pass x, slab edges,
slab fold, lower-envelope passes)."""

from __future__ import annotations

import numpy as np
import torch

import oracle

CLAMP = 255


def _np_view(t, dtype):
    return t.numpy().view(dtype)


def dist1d_axis0(occ: np.ndarray) -> np.ndarray:
    """1-D distance along axis 0 to the nearest True, clamped at 255."""
    out = np.empty(occ.shape, dtype=np.int64)
    run = np.full(occ.shape[1:], CLAMP, dtype=np.int64)
    for x in range(occ.shape[0]):
        run = np.where(occ[x], 0, np.minimum(run + 1, CLAMP))
        out[x] = run
    run = np.full(occ.shape[1:], CLAMP, dtype=np.int64)
    for x in range(occ.shape[0] - 1, -1, -1):
        run = np.where(occ[x], 0, np.minimum(run + 1, CLAMP))
        out[x] = np.minimum(out[x], run)
    return out


def cone_axis(g: np.ndarray, axis: int) -> np.ndarray:
    """out[i] = min(255, min_j max(|i - j|, g[j])) along one axis."""
    a = np.moveaxis(g.astype(np.int64), axis, -1)
    L = a.shape[-1]
    idx = np.arange(L)
    dist = np.abs(idx[:, None] - idx[None, :])
    out = np.maximum(dist, a[..., None, :]).min(axis=-1)
    return np.moveaxis(np.minimum(out, CLAMP), -1, axis)


class HostOps:
    def empty(self, shape, np_dtype):
        dt = {np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.int16,
              np.dtype(np.int32): torch.int32}[np.dtype(np_dtype)]
        return torch.zeros(tuple(int(s) for s in shape), dtype=dt)

    def voxels(self, volume):
        v = volume.voxels
        return torch.from_numpy(v.view(np.int16) if v.dtype == np.uint16 else v.copy())

    def plane(self, vol_t, x):
        return vol_t[x: x + 1].contiguous()

    def _dt(self, bits):
        return np.uint8 if bits == 8 else np.uint16

    def block_min_max(self, vol_t, bits, b):
        mn, mx = oracle.block_min_max(_np_view(vol_t, self._dt(bits)), b)
        as_t = (lambda a: torch.from_numpy(a.view(np.int16))) if bits == 16 else torch.from_numpy
        return as_t(mn), as_t(mx)

    def fold_minmax(self, mins_plane, maxs_plane, pmins, pmaxs, bits):
        dt = self._dt(bits)
        m, x = _np_view(mins_plane, dt), _np_view(maxs_plane, dt)
        np.minimum(m, _np_view(pmins, dt), out=m)
        np.maximum(x, _np_view(pmaxs, dt), out=x)

    def _bits_to_mask(self, on: np.ndarray, n: int) -> torch.Tensor:
        words = (n + 31) // 32
        mask = np.zeros((on.shape[1], words), dtype=np.uint32)
        for p in range(n):
            mask[on[p], p // 32] |= np.uint32(1 << (p % 32))
        return torch.from_numpy(mask.view(np.int32))

    def mask_from_minmax(self, mins, maxs, bits, scheme):
        dt = self._dt(bits)
        pid = scheme.pid_lut()
        plo = pid[_np_view(mins, dt).ravel().astype(np.int64)]
        phi = pid[_np_view(maxs, dt).ravel().astype(np.int64)]
        on = np.stack([(plo <= p) & (p <= phi) for p in range(scheme.n)])
        return self._bits_to_mask(on, scheme.n)

    def mask_voxel(self, vol_t, bits, b, scheme):
        pres = oracle.partition_presence(_np_view(vol_t, self._dt(bits)), b, scheme.pid_lut(),
                                         scheme.n)
        return self._bits_to_mask(pres.reshape(scheme.n, -1), scheme.n)

    def pass_x(self, mask, n, bdims, storage, pitch):
        m = mask.numpy().view(np.uint32)
        nb = int(np.prod(bdims))
        st = storage.numpy()
        for p in range(n):
            occ = ((m[:, p // 32] >> np.uint32(p % 32)) & 1).astype(bool).reshape(bdims)
            st[p, :nb] = dist1d_axis0(occ).ravel()

    def edges(self, storage, pitch, n, bdims):
        nb = int(np.prod(bdims))
        g = storage.numpy()[:, :nb].reshape((n,) + tuple(bdims))
        return torch.from_numpy(np.ascontiguousarray(np.stack([g[:, 0], g[:, -1]])))

    def fold(self, storage, pitch, n, bdims, edges_all, world, rank, slab_x0):
        """Restates slab_fold_kernel (csrc/dt.cu)."""
        nb = int(np.prod(bdims))
        bx = bdims[0]
        g = storage.numpy()[:, :nb].reshape((n,) + tuple(bdims)).astype(np.int64)
        e = edges_all.numpy().astype(np.int64)  # [world, 2, n, by, bz]
        big = 1 << 20
        below = np.full(e.shape[2:], big, dtype=np.int64)
        above = np.full(e.shape[2:], big, dtype=np.int64)
        my0, my1 = int(slab_x0[rank]), int(slab_x0[rank + 1])
        for j in range(world):
            if j < rank:
                hi = e[j, 1]
                below = np.minimum(below, np.where(hi < CLAMP, hi + my0 - int(slab_x0[j + 1]) + 1,
                                                   big))
            elif j > rank:
                lo = e[j, 0]
                above = np.minimum(above, np.where(lo < CLAMP, lo + int(slab_x0[j]) - my1 + 1,
                                                   big))
        x = np.arange(bx)[None, :, None, None]
        g = np.minimum(g, np.minimum(below[:, None] + x, CLAMP))
        g = np.minimum(g, np.minimum(above[:, None] + (bx - 1 - x), CLAMP))
        storage.numpy()[:, :nb] = g.reshape(n, nb).astype(np.uint8)

    def pass_yz(self, storage, pitch, n, bdims):
        nb = int(np.prod(bdims))
        g = storage.numpy()[:, :nb].reshape((n,) + tuple(bdims))
        g = cone_axis(cone_axis(g, 2), 3)
        storage.numpy()[:, :nb] = g.reshape(n, nb).astype(np.uint8)
