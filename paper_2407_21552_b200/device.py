"""Device-memory plumbing: numpy <-> CUDA tensors through pinned staging.

torch is used only as the allocator / stream / copy engine here; all compute
goes through libpdm_b200 kernels.  Host<->device copies go through pinned
(page-locked) buffers from torch's caching host allocator so they run at
full PCIe/C2C rate and are stream-ordered.
"""

from __future__ import annotations

import weakref

import numpy as np

PLANE_ALIGN = 256  # bytes between partition planes are a multiple of this
_PINNED_MIN = 1 << 16  # below this a plain pageable copy is cheaper


_TORCH = None


def torch():
    global _TORCH
    if _TORCH is None:
        import torch as _torch

        _TORCH = _torch
    return _TORCH


def device():
    from . import _lib

    _lib.lib()  # raises when no CUDA device / library: there is no CPU fallback
    return torch().device("cuda", torch().cuda.current_device())


_TORCH_DTYPE = {
    np.dtype(np.uint8): "uint8",
    np.dtype(np.uint16): "int16",  # reinterpreted: kernels only see raw bytes
    np.dtype(np.int16): "int16",
    np.dtype(np.int32): "int32",
    np.dtype(np.uint32): "int32",
    np.dtype(np.int64): "int64",
    np.dtype(np.float64): "float64",
    np.dtype(np.bool_): "uint8",
}
_VIEW_AS = {np.dtype(np.bool_): np.uint8, np.dtype(np.uint16): np.int16,
            np.dtype(np.uint32): np.int32}


_DT_CACHE: dict = {}


def _torch_dtype(dt):
    got = _DT_CACHE.get(dt)
    if got is None:
        got = _DT_CACHE[dt] = getattr(torch(), _TORCH_DTYPE[np.dtype(dt)])
    return got


def to_device(a: np.ndarray):
    """Upload a host array as raw bytes of the same shape (stream-ordered)."""
    t = torch()
    dev = device()
    a = np.ascontiguousarray(a)
    dt = np.dtype(a.dtype)
    src = t.from_numpy(a.view(_VIEW_AS[dt]) if dt in _VIEW_AS else a)
    if a.nbytes >= _PINNED_MIN:
        staged = t.empty(src.shape, dtype=src.dtype, pin_memory=True)
        staged.copy_(src)
        # non_blocking from pinned memory: torch's caching host allocator holds
        # `staged` until the copy has completed on the current stream
        return staged.to(dev, non_blocking=True)
    return src.to(dev)


def to_host(t_dev, np_dtype) -> np.ndarray:
    """Download a device tensor into pinned host memory; reinterpret as np_dtype."""
    t = torch()
    np_dtype = np.dtype(np_dtype)
    if t_dev.numel() * t_dev.element_size() >= _PINNED_MIN:
        host_t = t.empty(t_dev.shape, dtype=t_dev.dtype, pin_memory=True)
        host_t.copy_(t_dev, non_blocking=True)
        t.cuda.current_stream().synchronize()
    else:
        host_t = t_dev.detach().to("cpu")
    host = host_t.numpy()
    if np_dtype == np.bool_:
        return host.astype(bool)
    if host.dtype.itemsize == np_dtype.itemsize:
        return host.view(np_dtype)
    return host.astype(np_dtype)


def complete() -> None:
    """Wait for the current stream: the public API returns completed results,
    as the reference's synchronous numpy/numba functions do, so a caller's own
    timer (bench.measure_ms, SessionStore.set_tf) measures the device work."""
    from . import _lib

    _lib.check(_lib.lib().pdm_stream_synchronize(_lib.stream_handle()), "stream synchronize")


_EMPTY = None


def empty(shape, np_dtype):
    """Uninitialised tensor on the current CUDA device (raises without one)."""
    global _EMPTY
    if _EMPTY is None:
        from . import _lib

        _lib.lib()  # no CUDA device / library: there is no CPU fallback
        _EMPTY = torch().empty
    dt = _DT_CACHE.get(np_dtype)
    if dt is None:
        dt = _torch_dtype(np_dtype)
    return _EMPTY(shape, dtype=dt, device="cuda")


def plane_pitch(num_blocks: int) -> int:
    return -(-int(num_blocks) // PLANE_ALIGN) * PLANE_ALIGN


# ---- recycled host result buffers ---------------------------------------------------
# Host views of device results (e.g. D' expanded on the host) land in pageable
# buffers recycled per size: a fresh large numpy array pays its page faults
# (and the kernel's page zeroing) on first touch -- ~6 ms for a 134 MB map --
# while a recycled one is already mapped.  Ownership is explicit: each array
# handed out is a view of a _PoolBlock (numpy keeps the block as the .base of
# every view and slice made from it), and the block's finalizer returns the
# raw buffer to the pool only when the last of those arrays is gone.
_HOST_POOL: dict = {}
_HOST_POOL_CAP = 4  # idle buffers kept per size


class _PoolBlock:
    """Buffer exporter owning one pooled raw buffer (PEP 688 __buffer__)."""

    __slots__ = ("raw", "__weakref__")

    def __init__(self, raw: np.ndarray):
        self.raw = raw

    def __buffer__(self, flags):
        return memoryview(self.raw)


def _recycle(nbytes: int, raw: np.ndarray) -> None:
    pool = _HOST_POOL.setdefault(nbytes, [])
    if len(pool) < _HOST_POOL_CAP:
        pool.append(raw)


def host_buffer(shape) -> np.ndarray:
    """A writable, 64-byte aligned uint8 array of `shape` backed by a recycled
    buffer (returned to the pool once no array references it)."""
    nbytes = int(np.prod(shape))
    pool = _HOST_POOL.setdefault(nbytes, [])
    raw = pool.pop() if pool else np.empty(nbytes + 64, dtype=np.uint8)
    blk = _PoolBlock(raw)
    weakref.finalize(blk, _recycle, nbytes, raw)
    flat = np.frombuffer(blk, dtype=np.uint8)
    off = (-flat.ctypes.data) % 64  # the host expansion streams whole cache lines
    return flat[off:off + nbytes].reshape(shape)
