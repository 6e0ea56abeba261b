"""Where the full recompute (standard_distance_map, the Deakin baseline and the
block-ESS row of the paper's Fig. 4) spends its time at BASELINE config c.

Times each stage through the C ABI with CUDA events on the launching stream
(median of --reps after warm-up), and the whole public call.

    python tools/recompute_probe.py [--dims 1024 1024 1024] [--b 4] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import _lib, device, synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[1024, 1024, 1024])
    ap.add_argument("--bits", type=int, default=16)
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    L = _lib.lib()
    st = _lib.stream_handle()
    stream = torch.cuda.current_stream()
    vol = synth.synth_volume_device(tuple(args.dims), args.bits, seed=2407, nbox=12)
    grid = pdm.BlockGrid.for_dims(vol.dims, args.b)
    bx, by, bz = grid.bdims
    nb = grid.num_blocks

    def timed(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return round(float(np.median(ts)), 4)

    tf = pdm.tf_archetype("tf3", args.bits)
    res = {"dims": args.dims, "bits": args.bits, "b": args.b, "blocks": nb}
    occ = pdm.occupancy_for_tf(vol, grid, tf)
    occ_dev = occ.device()
    out = device.empty((nb,), np.uint8)
    mm = pdm.block_min_max_device(vol, grid)
    res["occupancy_for_tf_voxel_ms"] = timed(lambda: pdm.occupancy_for_tf(vol, grid, tf))
    res["occupancy_for_tf_range_apron_ms"] = timed(
        lambda: pdm.occupancy_for_tf(vol, grid, tf, "range_apron"))
    res["occupancy_for_tf_minmax_given_ms"] = timed(
        lambda: pdm.occupancy_for_tf(vol, grid, tf, "range_apron", minmax=mm))
    res["block_min_max_ms"] = timed(lambda: pdm.block_min_max_device(vol, grid))

    def dt():
        _lib.check(L.pdm_distance_transform(_lib.ptr(occ_dev), bx, by, bz, _lib.ptr(out), st),
                   "dt")
    res["distance_transform_abi_ms"] = timed(dt)
    res["distance_transform_api_ms"] = timed(lambda: pdm.distance_transform(occ))
    for m in ("voxel", "range_apron"):
        res[f"standard_distance_map_{m}_ms"] = timed(
            lambda: pdm.standard_distance_map(vol, grid, tf, m))
    res["standard_distance_map_minmax_given_ms"] = timed(
        lambda: pdm.standard_distance_map(vol, grid, tf, "range_apron", minmax=mm))
    res["volume_roofline_ms"] = round(vol.nbytes / 6553.3e9 * 1e3, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
