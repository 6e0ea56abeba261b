"""All BASELINE.json configs on one B200 (bench.py covers config c).

    python tools/configs_bench.py [--configs a b d e] [--cpu]

a: 256^3 uint8, b=4, n=8, random 1-D TF changes (tf_from_support, p in
   {0.02, 0.1, 0.5}) -- select+merge vs full recompute (voxel and range_apron)
b: 512^3 uint16, b=8, n=16 -- PDM merge vs full occupancy + Chebyshev recompute
d: 2048^3 uint16, b=4, n=32 on ONE GPU (17.2 GB volume) -- precompute + merge
e: 1024^3 uint16, b=4, n in {4,8,16,32,64} -- PDM footprint vs update latency

Device timings are CUDA events (median of reps, L2 flushed before each rep);
`api_ms` is the public API with host buffers (select_partitions + combine +
.dist); `cpu_ms` is the C oracle (all host threads) on the same bytes.
Prints one JSON line per config.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["a", "b", "e", "d"])
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--cpu", action="store_true", help="also time the C oracle")
    args = ap.parse_args()
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_r = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")

    class flush:  # write 256 MB then read 256 MB: L2 emptied, dirty lines drained
        @staticmethod
        def fill_(v):
            flush_w.fill_(v)
            flush_r.sum()

    def dev_ms(fn):
        ts = []
        for r in range(args.reps + 2):
            flush.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        return round(float(np.median(ts)), 4)

    def wall_ms(fn, reps=None):
        ts = []
        for r in range((reps or args.reps) + 1):
            flush.fill_(r & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            if r >= 1:
                ts.append((time.perf_counter() - t0) * 1e3)
        return round(float(np.median(ts)), 4)

    def aligned_alpha(scheme, k, rng):
        span = scheme.intensity_span
        alpha = np.zeros(span)
        for p in rng.choice(scheme.n, size=k, replace=False):
            part = scheme.partitions[p]
            alpha[part.rho_lo: part.rho_hi + 1] = rng.uniform(0.05, 1.0, part.width)
        return alpha

    def tf_of(alpha):
        lut = np.zeros((alpha.size, 4))
        lut[:, 3] = alpha
        return pdm.TransferFunction(lut=lut)

    def update_row(pset, vol, grid, scheme, tf, label, cpu=False):
        alpha_dev = torch.from_numpy(np.ascontiguousarray(tf.lut[:, 3])).cuda()
        out = torch.empty(grid.bdims, dtype=torch.uint8, device="cuda")
        flags = torch.empty(scheme.n, dtype=torch.uint8, device="cuda")
        sel = pdm.select_partitions(tf, scheme)
        k = len(sel)
        row = {"tf": label, "k": k,
               "update_ms": dev_ms(lambda: pdm.update_from_tf(pset, alpha_dev, out, flags)),
               "api_ms": wall_ms(lambda: pdm.combine(pset, pdm.select_partitions(tf, scheme)).dist),
               "recompute_voxel_ms": dev_ms(lambda: pdm.standard_distance_map(vol, grid, tf)),
               "recompute_range_apron_ms": dev_ms(
                   lambda: pdm.standard_distance_map(vol, grid, tf, "range_apron"))}
        row["merge_bytes"] = (k + 1) * grid.num_blocks
        row["update_GBps"] = round(row["merge_bytes"] / row["update_ms"] / 1e6, 1)
        row["speedup_vs_recompute_voxel"] = round(row["recompute_voxel_ms"] / row["update_ms"], 1)
        assert np.array_equal(pdm.combine(pset, sel).dist, out.cpu().numpy())
        if cpu:
            import oracle

            oracle.set_threads(oracle.max_threads())
            nb = grid.num_blocks
            maps = pset.storage[:, :nb].cpu().numpy()
            bounds = scheme.bounds()
            a = np.ascontiguousarray(tf.lut[:, 3])
            t0 = time.perf_counter()
            for _ in range(3):
                oracle.combine(maps, oracle.select(a, bounds))
            row["cpu_update_ms"] = round((time.perf_counter() - t0) / 3 * 1e3, 3)
            row["cpu_threads"] = oracle.max_threads()
        return row

    def build(dims, bits, b, n, seed):
        vol = synth.synth_volume_device(dims, bits, seed=seed, nbox=12)
        grid = pdm.BlockGrid.for_dims(dims, b)
        scheme = pdm.scheme_uniform(n, bits)
        pset = pdm.build_pdm_set(vol, grid, scheme)  # warm (first call pays lazy init)
        t = {m: dev_ms(lambda: pdm.build_pdm_set(vol, grid, scheme, m))
             for m in ("voxel", "range_apron")}
        return vol, grid, scheme, pset, t

    rng = np.random.default_rng(2407)
    for cfg in args.configs:
        if cfg == "a":
            vol, grid, scheme, pset, t = build((256, 256, 256), 8, 4, 8, 11)
            rows = []
            for p in (0.02, 0.1, 0.5):
                support = rng.random(256) < p
                lut = np.zeros((256, 4))
                lut[support, 3] = rng.uniform(0.05, 1.0, support.sum())
                rows.append(update_row(pset, vol, grid, scheme, pdm.TransferFunction(lut=lut),
                                       f"random p={p}", args.cpu))
            print(json.dumps({"config": "a: 256^3 u8, b=4, n=8, random 1-D TF changes",
                              "precompute_ms": t, "rows": rows}), flush=True)
        elif cfg == "b":
            vol, grid, scheme, pset, t = build((512, 512, 512), 16, 8, 16, 12)
            rows = [update_row(pset, vol, grid, scheme, tf_of(aligned_alpha(scheme, k, rng)),
                               f"aligned k={k}", args.cpu) for k in (4, 16)]
            rows.append(update_row(pset, vol, grid, scheme, pdm.tf_archetype("tf3", 16), "tf3",
                                   args.cpu))
            print(json.dumps({"config": "b: 512^3 u16, b=8, n=16, merge vs full recompute",
                              "precompute_ms": t, "rows": rows}), flush=True)
        elif cfg == "e":
            vol = synth.synth_volume_device((1024, 1024, 1024), 16, seed=2407, nbox=12)
            grid = pdm.BlockGrid.for_dims(vol.dims, 4)
            rows = []
            for n in (4, 8, 16, 32, 64):
                scheme = pdm.scheme_uniform(n, 16)
                pset = pdm.build_pdm_set(vol, grid, scheme)
                pre = dev_ms(lambda: pdm.build_pdm_set(vol, grid, scheme))
                r_all = update_row(pset, vol, grid, scheme, tf_of(aligned_alpha(scheme, n, rng)),
                                   f"aligned k={n}")
                r_half = update_row(pset, vol, grid, scheme,
                                    tf_of(aligned_alpha(scheme, max(1, n // 2), rng)),
                                    f"aligned k={max(1, n // 2)}")
                rows.append({"n": n, "pdm_bytes": pset.memory_bytes(),
                             "device_bytes": pset.device_bytes(),  # raw + packed + tile bounds
                             "precompute_ms": pre,
                             "update_ms_k_n": r_all["update_ms"],
                             "update_GBps_k_n": r_all["update_GBps"],
                             "update_ms_k_half": r_half["update_ms"],
                             "recompute_voxel_ms": r_all["recompute_voxel_ms"]})
                del pset
                torch.cuda.empty_cache()
            print(json.dumps({"config": "e: 1024^3 u16, b=4, partition-count sweep",
                              "rows": rows}), flush=True)
        elif cfg == "d":
            vol, grid, scheme, pset, t = build((2048, 2048, 2048), 16, 4, 32, 13)
            rows = [update_row(pset, vol, grid, scheme, tf_of(aligned_alpha(scheme, k, rng)),
                               f"aligned k={k}") for k in (1, 16, 32)]
            print(json.dumps({"config": "d: 2048^3 u16, b=4, n=32 on one B200 (17.2 GB volume)",
                              "precompute_ms": t, "rows": rows}), flush=True)
            del vol, pset
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
