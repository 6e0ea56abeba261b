"""Live TF-edit session on the device.

Mirrors /root/reference/pkg/src/pdmrender/service/session.py:60-127
(``SessionStore.load`` / ``snapshot`` / ``set_tf``) with the PDM set and every
combined map resident in HBM: ``set_tf`` selects and merges on the GPU
(select_partitions_device + combine_flags_into, no host round trip), times
both with CUDA events, and reports the combined map's occupied fraction (the
service's ``dprime_nonzero_fraction``, service/app.py:129) from a zero count
the merge kernel keeps while it writes D' (packed sets; a separate count
kernel otherwise), so an edit moves 8 bytes back to the host instead of the
16.8 MB map.
The (tf, selection, dprime) triple is swapped under a lock like the
reference; readers holding an older snapshot keep a valid map because every
update writes a fresh buffer.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np

from . import device
from .acceleration import DistanceMap, PdmSet, build_pdm_set, combine_flags_into
from .transfer import (
    PartitionScheme,
    PartitionSelection,
    TransferFunction,
    alpha_to_device,
    select_partitions_device,
)
from .volume import BlockGrid, Volume


class NoSessionError(RuntimeError):
    """No volume loaded yet (service/session.py:37)."""


@dataclass(frozen=True)
class Session:
    volume: Volume
    grid: BlockGrid
    scheme: PartitionScheme
    pdm_set: PdmSet
    occupancy_mode: str
    tf: TransferFunction
    selection: PartitionSelection
    dprime: DistanceMap
    select_ms: float
    combine_ms: float
    dprime_occupied_fraction: float = 0.0
    wall_ms: float = 0.0


def _empty_tf(bits: int) -> TransferFunction:
    return TransferFunction(lut=np.zeros((1 << bits, 4)))


class PdmSessionStore:
    """One live session (the reference's SessionStore) on the GPU."""

    def __init__(self) -> None:
        self._lock = threading.Lock()
        self._session: Session | None = None

    def load(self, volume: Volume, grid: BlockGrid, scheme: PartitionScheme,
             occupancy_mode: str = "range_apron") -> Session:
        pdm_set = build_pdm_set(volume, grid, scheme, occupancy_mode)
        tf = _empty_tf(volume.bits)
        session = self._update(volume, grid, scheme, pdm_set, occupancy_mode, tf)
        session = Session(**{**session.__dict__, "select_ms": 0.0, "combine_ms": 0.0})
        with self._lock:
            self._session = session
        return session

    def snapshot(self) -> Session:
        with self._lock:
            if self._session is None:
                raise NoSessionError("no volume loaded")
            return self._session

    def set_tf(self, tf: TransferFunction) -> Session:
        with self._lock:
            if self._session is None:
                raise NoSessionError("no volume loaded")
            base = self._session
        if tf.bits != base.volume.bits:
            raise ValueError(f"transfer function is {tf.bits}-bit, session volume needs "
                             f"{base.volume.bits}-bit")
        session = self._update(base.volume, base.grid, base.scheme, base.pdm_set,
                               base.occupancy_mode, tf)
        with self._lock:
            self._session = session
        return session

    @staticmethod
    def _update(volume, grid, scheme, pdm_set, mode, tf) -> Session:
        torch = device.torch()
        t_wall = time.perf_counter()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        flags = select_partitions_device(alpha_to_device(tf), scheme)
        ev[1].record()
        dprime = combine_flags_into(pdm_set, flags, count_zeros=True)
        ev[2].record()
        occupied = dprime.occupied_fraction  # zero count from the merge; synchronises
        wall_ms = (time.perf_counter() - t_wall) * 1e3
        return Session(volume=volume, grid=grid, scheme=scheme, pdm_set=pdm_set,
                       occupancy_mode=mode, tf=tf,
                       selection=PartitionSelection(n=scheme.n, flags_dev=flags), dprime=dprime,
                       select_ms=ev[0].elapsed_time(ev[1]), combine_ms=ev[1].elapsed_time(ev[2]),
                       dprime_occupied_fraction=occupied, wall_ms=wall_ms)
