"""Where a small-map TF update spends its time through the public API (the
reference acceptance check's 256^3 u8, b=4, n=64, 16 selected): every piece
of select_partitions and combine timed on its own (median of 200)."""
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2407_21552_b200 as P  # noqa: E402
from paper_2407_21552_b200 import _lib, device  # noqa: E402


def med(fn, reps=200):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(ts), 2)


def main():
    rng = np.random.default_rng(7)
    vox = rng.integers(0, 256, size=(256, 256, 256), dtype=np.uint8)
    vox[vox < 200] = 0
    vol = P.Volume.from_array(vox)
    grid = P.BlockGrid.for_dims(vol.dims, 4)
    lut = np.zeros((256, 4))
    lut[128:192, 3] = 0.5
    tf = P.TransferFunction(lut=lut)
    scheme = P.scheme_uniform(64, bits=8)
    pset = P.build_pdm_set(vol, grid, scheme, "voxel")
    sel = P.select_partitions(tf, scheme)
    L = _lib.lib()
    st = _lib.stream_handle()
    stg = scheme._select_stage(st)
    r = {}
    r["select_partitions"] = med(lambda: P.select_partitions(tf, scheme))
    r["pdm_select_tf (ctypes, gather+launch+sync)"] = med(lambda: L.pdm_select_tf(
        lut.ctypes.data + 24, 256, 4, stg.host_ptr, stg.dev_ptr, stg.starts_ptr, 64,
        scheme.max_width, stg.flags_dev_ptr, stg.flags_host_ptr, st))
    r["select: stream_handle"] = med(lambda: _lib.stream_handle())
    r["select: flatnonzero+frozenset+obj"] = med(lambda: P.PartitionSelection._from_checked(
        frozenset((np.flatnonzero(stg.flags_host) + 1).tolist()), 64))
    r["combine"] = med(lambda: P.combine(pset, sel))
    idx = np.ascontiguousarray([i - 1 for i in sel.sorted], dtype=np.int32)
    out = device.empty(grid.bdims, np.uint8)
    args = pset._packed_args()
    r["combine: sorted+int32 array"] = med(lambda: np.ascontiguousarray(
        [i - 1 for i in sel.sorted], dtype=np.int32))
    r["combine: device.empty"] = med(lambda: device.empty(grid.bdims, np.uint8))
    r["combine: DistanceMap()"] = med(lambda: P.DistanceMap(b=4, bdims=grid.bdims, dist=out))

    def launch():
        L.pdm_combine_packed(*args, grid.num_blocks, 64, idx.ctypes.data, int(idx.size),
                             out.data_ptr(), None, st)
    r["combine: pdm_combine_packed launch (+sync outside)"] = med(
        lambda: (launch(), L.pdm_stream_synchronize(st)))
    r["stream sync idle"] = med(lambda: L.pdm_stream_synchronize(st))
    r["update = combine(select(...))"] = med(lambda: P.combine(pset, P.select_partitions(tf, scheme)))
    r["rebuild standard_distance_map voxel"] = med(
        lambda: P.standard_distance_map(vol, grid, tf, "voxel"), 50)
    r["ratio"] = round(r["rebuild standard_distance_map voxel"] / r["update = combine(select(...))"], 2)
    print(json.dumps(r, indent=1))


if __name__ == "__main__" and "--c" not in sys.argv:
    main()


def c_floor():
    """C-level pieces of one round trip (ctypes calls, median of 300)."""
    import torch

    L = _lib.lib()
    st = _lib.stream_handle()
    span, n = 256, 64
    alpha_dev = torch.zeros(span, dtype=torch.float64, device="cuda")
    alpha_dev[128:192] = 0.5
    flags_dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    alpha_pin = torch.zeros(span, dtype=torch.float64, pin_memory=True)
    alpha_pin[128:192] = 0.5
    flags_pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    tiny = torch.zeros(16, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    r = {}
    r["count_value(16 B)+sync (floor)"] = med(lambda: (L.pdm_count_value(
        tiny.data_ptr(), 16, 0, cnt.data_ptr(), st), L.pdm_stream_synchronize(st)), 300)
    r["select dev alpha/dev flags +sync"] = med(lambda: (L.pdm_select(
        alpha_dev.data_ptr(), span, 1, None, n, 4, flags_dev.data_ptr(), st),
        L.pdm_stream_synchronize(st)), 300)
    r["select zero-copy alpha/flags +sync"] = med(lambda: (L.pdm_select(
        alpha_pin.data_ptr(), span, 1, None, n, 4, flags_pin.data_ptr(), st),
        L.pdm_stream_synchronize(st)), 300)
    r["select launch only (no sync)"] = med(lambda: L.pdm_select(
        alpha_dev.data_ptr(), span, 1, None, n, 4, flags_dev.data_ptr(), st), 300)
    L.pdm_stream_synchronize(st)
    print(json.dumps(r, indent=1))


if __name__ == "__main__" and "--c" in sys.argv:
    c_floor()
