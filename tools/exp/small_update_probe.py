"""Where the time of a small-map TF update goes through the public API
(the reference acceptance check test_acceptance.py:349-392: 256^3 u8 sphere
shell, b=4, n=64, 16 partitions selected; update must beat the full rebuild
3x under the reference's own perf_counter timer, bench.py:192-200)."""

import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2407_21552_b200 as P  # noqa: E402
from paper_2407_21552_b200 import _lib  # noqa: E402


def med(fn, reps=50):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 4)


def main():
    import torch

    rng = np.random.default_rng(7)
    vox = rng.integers(0, 256, size=(256, 256, 256), dtype=np.uint8)
    vox[vox < 200] = 0
    vol = P.Volume.from_array(vox)
    grid = P.BlockGrid.for_dims(vol.dims, 4)
    support = np.zeros(256, dtype=bool)
    support[128:192] = True
    lut = np.zeros((256, 4))
    lut[support, 3] = 0.5
    tf = P.TransferFunction(lut=lut)
    scheme = P.scheme_uniform(64, bits=8)
    pset = P.build_pdm_set(vol, grid, scheme, "voxel")
    sel = P.select_partitions(tf, scheme)
    L = _lib.lib()
    st = _lib.stream_handle()
    out = {}
    out["ctypes_version"] = med(lambda: L.pdm_version())
    out["stream_sync_idle"] = med(lambda: L.pdm_stream_synchronize(st))
    out["torch_sync_idle"] = med(lambda: torch.cuda.synchronize())
    out["empty_alloc"] = med(lambda: P.device.empty(grid.bdims, np.uint8))
    out["select"] = med(lambda: P.select_partitions(tf, scheme))
    out["combine"] = med(lambda: P.combine(pset, sel))
    out["update"] = med(lambda: P.combine(pset, P.select_partitions(tf, scheme)))
    out["rebuild_voxel"] = med(lambda: P.standard_distance_map(vol, grid, tf, "voxel"))
    out["ratio"] = round(out["rebuild_voxel"] / out["update"], 2)
    # device-only times
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()

    def dev(fn, reps=30):
        ts = []
        for _ in range(reps):
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return round(statistics.median(ts), 4)

    out["dev_combine"] = dev(lambda: P.combine(pset, sel))
    out["dev_rebuild"] = dev(lambda: P.standard_distance_map(vol, grid, tf, "voxel"))
    print(json.dumps(out))


if __name__ == "__main__" and "--breakdown" not in sys.argv:
    main()


def breakdown():
    """Sub-steps of combine() / select_partitions() at the acceptance config."""
    import torch

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
    acc = P.acceleration
    idx = np.ascontiguousarray([i - 1 for i in sel.sorted], dtype=np.int32)
    out_t = P.device.empty(grid.bdims, np.uint8)
    nib, nib_pitch, base, base_pitch = pset.packed()
    r = {}
    r["sorted+array"] = med(lambda: np.ascontiguousarray([i - 1 for i in sel.sorted],
                                                         dtype=np.int32))
    r["stream_handle"] = med(lambda: _lib.stream_handle())
    r["packed()"] = med(lambda: pset.packed())
    st = _lib.stream_handle()

    def launch_only():
        L.pdm_combine_packed(_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                             pset.tile_bounds_ptr(), grid.num_blocks, pset.n, idx.ctypes.data, int(idx.size),
                             _lib.ptr(out_t), None, st)

    def launch_sync():
        launch_only()
        L.pdm_stream_synchronize(st)

    r["launch_only(+drain)"] = med(lambda: (launch_only(), torch.cuda.synchronize()))
    r["launch_sync"] = med(launch_sync)
    r["_combine_indices+complete"] = med(lambda: (acc._combine_indices(pset, idx, out_t),
                                                  P.device.complete()))
    r["DistanceMap()"] = med(lambda: P.DistanceMap(b=4, bdims=grid.bdims, dist=out_t))
    r["combine"] = med(lambda: P.combine(pset, sel))
    stg = scheme._select_stage(st)
    r["select_tf_c"] = med(lambda: L.pdm_select_tf(lut.ctypes.data + 24, 256, 4, stg.host_ptr,
                                                   stg.dev_ptr, stg.starts_ptr, 64,
                                                   scheme.max_width, stg.flags_dev_ptr,
                                                   stg.flags_host_ptr, st))
    r["select"] = med(lambda: P.select_partitions(tf, scheme))
    r["rebuild_voxel"] = med(lambda: P.standard_distance_map(vol, grid, tf, "voxel"))
    print(json.dumps(r))
    from torch.profiler import ProfilerActivity, profile

    for name, fn in (("combine", lambda: P.combine(pset, sel)),
                     ("select", lambda: P.select_partitions(tf, scheme)),
                     ("rebuild", lambda: P.standard_distance_map(vol, grid, tf, "voxel"))):
        fn()
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for _ in range(20):
                fn()
        print("=====", name)
        print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=25,
                                        max_name_column_width=60))


if __name__ == "__main__" and "--breakdown" in sys.argv:
    breakdown()
