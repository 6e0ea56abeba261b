"""PDM precompute stages at BASELINE config c (1024^3 u16, b=4, n=32) and the
full-recompute baseline (standard_distance_map), timed with CUDA events.

    python tools/precompute_bench.py [--dims 1024 1024 1024] [--n 32] [--b 4]
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
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    L = _lib.lib()
    st = _lib.stream_handle()
    vol = synth.synth_volume_device(tuple(args.dims), args.bits, seed=2407, nbox=12)
    grid = pdm.BlockGrid.for_dims(vol.dims, args.b)
    scheme = pdm.scheme_uniform(args.n, args.bits)
    nb = grid.num_blocks
    vbytes = vol.nbytes

    def timed(fn):
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return round(min(ts), 4)

    res = {"dims": args.dims, "bits": args.bits, "b": args.b, "n": args.n, "blocks": nb}
    pitch = device.plane_pitch(nb)
    storage = device.empty((args.n, pitch), np.uint8)
    for mode in ("voxel", "range_apron"):
        mask = pdm.partition_mask(vol, grid, scheme, mode)
        ms = timed(lambda: pdm.partition_mask(vol, grid, scheme, mode))
        res[f"mask_{mode}_ms"] = ms
        res[f"mask_{mode}_GBps"] = round((vbytes + nb * 4) / ms / 1e6, 1)
        res[f"dt_pass_x_{mode}_ms"] = timed(lambda: _lib.check(L.pdm_dt_pass_x_mask(
            _lib.ptr(mask), mask.shape[1], args.n, *grid.bdims, _lib.ptr(storage), pitch, st),
            "pass_x"))
    words = mask.shape[1]

    def pass_x():
        _lib.check(L.pdm_dt_pass_x_mask(_lib.ptr(mask), words, args.n, *grid.bdims,
                                        _lib.ptr(storage), pitch, st), "pass_x")

    def pass_yz():
        _lib.check(L.pdm_dt_pass_yz(_lib.ptr(storage), pitch, args.n, *grid.bdims, st), "yz")

    res["dt_pass_x_ms"] = timed(pass_x)
    pass_x()
    res["dt_pass_yz_ms"] = timed(lambda: (pass_x(), pass_yz())) - res["dt_pass_x_ms"]
    res["build_pdm_set_ms"] = {m: timed(lambda: pdm.build_pdm_set(vol, grid, scheme, m))
                               for m in ("voxel", "range_apron")}
    tf = pdm.tf_archetype("tf3", args.bits)
    res["standard_distance_map_ms"] = {
        m: timed(lambda: pdm.standard_distance_map(vol, grid, tf, m)) for m in ("voxel",
                                                                                 "range_apron")}
    res["block_min_max_ms"] = timed(lambda: pdm.block_min_max_device(vol, grid))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
