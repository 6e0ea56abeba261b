"""Merge (K7) micro-benchmark: achieved HBM GB/s of pdm_combine vs k.

    python tools/merge_microbench.py [--blocks 16777216] [--n 32] [--reps 20]

Random PDM bytes (the merge is data-independent), L2 flushed before every
timed launch, CUDA events on the launching stream.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2407_21552_b200 import _lib, device

    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=256 ** 3)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    L = _lib.lib()
    nb, n = args.blocks, args.n
    pitch = device.plane_pitch(nb)
    pdms = torch.randint(0, 256, (n, pitch), dtype=torch.uint8, device="cuda")
    out = torch.empty(nb, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = _lib.stream_handle()
    res = {}
    for k in (1, 2, 4, 8, 16, 24, 32):
        if k > n:
            break
        sel = np.ascontiguousarray(np.arange(k), dtype=np.int32)
        ts = []
        for r in range(args.reps + 3):
            flush.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(L.pdm_combine(_lib.ptr(pdms), pitch, nb, n, sel.ctypes.data, k,
                                     _lib.ptr(out), st), "pdm_combine")
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        gbs = (k + 1) * nb / (ms * 1e-3) / 1e9
        res[k] = {"ms": round(ms, 5), "GB/s": round(gbs, 1)}
        want = pdms[:k, :nb].min(dim=0).values
        assert torch.equal(out, want)
    print(json.dumps({"blocks": nb, "n": n, "merge": res}))


if __name__ == "__main__":
    main()
