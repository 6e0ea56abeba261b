"""Frame time of the GPU ray marcher consuming D' in HBM
at config c, against the same marcher without skipping and against the C
restatement of the reference marcher (oracle/march_oracle.c, all host
threads) on a bounded sample of the same rays.

    python tools/render_bench.py [--size 1024] [--reps 10] [--cpu-rows 32]

Prints one JSON line.  Ray generation + marching are timed with CUDA events
on the launching stream (warm, median of --reps); `render_api_ms` adds the
framebuffer download (render() as a caller sees it).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, default=1024)
    ap.add_argument("--size", type=int, default=1024, help="viewport edge (pixels)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--k", type=int, default=8, help="partitions the TF selects")
    ap.add_argument("--cpu-rows", type=int, default=32, help="scanlines timed on the CPU")
    args = ap.parse_args()

    import torch

    import oracle
    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import raycast, synth

    dims = (args.dims,) * 3
    vol = synth.synth_volume_device(dims, 16, seed=2407, nbox=12)
    grid = pdm.BlockGrid.for_dims(dims, 4)
    scheme = pdm.scheme_uniform(32, 16)
    pset = pdm.build_pdm_set(vol, grid, scheme)
    rng = np.random.default_rng(5)
    picks = sorted(rng.choice(np.arange(1, 33), size=args.k, replace=False).tolist())
    lut = np.zeros((1 << 16, 4))
    for i in picks:
        p = scheme.partitions[i - 1]
        t = np.linspace(0.0, 1.0, p.rho_hi - p.rho_lo + 1)
        lut[p.rho_lo: p.rho_hi + 1] = np.stack([t, 1 - t, 0.5 + 0 * t, 0.02 + 0.05 * t], 1)
    tf = pdm.TransferFunction(lut=lut)
    dprime = pdm.combine(pset, pdm.select_partitions(tf, scheme))
    cam = pdm.orbit_camera(vol, angle=0.6)
    out = {"config": f"c: {args.dims}^3 u16 volume, b=4, n=32, TF selecting k={args.k} "
                     f"partitions, {args.size}x{args.size} viewport, step 0.5, ERT 0.98",
           "data": "synthetic (device-born banded boxes), orbit camera angle 0.6"}
    stream = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    for mode, accel in (("none", None), ("pdm", dprime)):
        st = pdm.RenderSettings(args.size, args.size, step=0.5, ess_mode=mode)
        ms = timed(lambda: raycast._march(vol, tf, cam, st, accel))
        api = []
        for _ in range(5):
            t0 = time.perf_counter()
            fb, stats = pdm.render(vol, tf, cam, st, accel)
            api.append((time.perf_counter() - t0) * 1e3)
        api_ms = float(np.median(api))
        total = stats.samples_evaluated + stats.samples_skipped
        out[mode] = {"frame_ms": round(ms, 3), "render_api_ms": round(api_ms, 3),
                     "samples_total": total, "samples_evaluated": stats.samples_evaluated,
                     "skip_events": stats.blocks_skipped, "ert": stats.ert_terminations,
                     "fixed_grid_Gsamples_per_s": round(total / (ms * 1e-3) / 1e9, 2),
                     "evaluated_Gsamples_per_s": round(stats.samples_evaluated / (ms * 1e-3) / 1e9,
                                                       2)}
        if mode == "pdm":
            pix_pdm = fb.pixels
        else:
            pix_none = fb.pixels
    out["pdm_identical_to_none"] = bool(np.array_equal(pix_pdm, pix_none))
    out["pdm_speedup_vs_none"] = round(out["none"]["frame_ms"] / out["pdm"]["frame_ms"], 2)

    # TF change -> new frame: D' update (select + merge) + march, device-resident
    st = pdm.RenderSettings(args.size, args.size, step=0.5, ess_mode="pdm")
    out["tf_change_to_frame_ms"] = round(timed(lambda: raycast._march(
        vol, tf, cam, st, pdm.combine(pset, pdm.select_partitions(tf, scheme)))), 3)

    # CPU: the oracle marcher on every (size / cpu_rows)-th scanline of the same rays
    threads = oracle.max_threads()
    oracle.set_threads(threads)
    origin, dirs = pdm.camera_rays(cam, args.size, args.size, vol)
    rows = np.linspace(0, args.size - 1, args.cpu_rows).astype(int)
    sample = np.ascontiguousarray(dirs.reshape(args.size, args.size, 3)[rows].reshape(-1, 3))
    vox = vol.voxels
    d_host = dprime.dist
    t0 = time.perf_counter()
    rgba, counters = oracle.march_rays(vox, lut, d_host, 4, 0.5, True, 0.98, origin, sample)
    cpu_s = time.perf_counter() - t0
    gpu_rgba = raycast._march(vol, tf, cam, st, dprime, per_ray=True)[2].cpu().numpy()
    gpu_rows = gpu_rgba.reshape(args.size, args.size, 4)[rows].reshape(-1, 4)
    out["cpu_baseline"] = {
        "kind": "port", "cores": threads,
        "sample": f"{len(rows)} of {args.size} scanlines ({sample.shape[0]} rays), pdm skipping",
        "rays_per_s": round(sample.shape[0] / cpu_s),
        "frame_ms_estimate": round(cpu_s * args.size / len(rows) * 1e3, 1),
        "bit_identical_to_gpu": bool(np.array_equal(rgba.view(np.uint64),
                                                    gpu_rows.view(np.uint64)))}
    out["gpu_speedup_vs_cpu_pdm"] = round(out["cpu_baseline"]["frame_ms_estimate"]
                                          / out["pdm"]["frame_ms"], 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
