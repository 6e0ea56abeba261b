"""Merge (K7) micro-benchmark: achieved HBM GB/s of pdm_combine vs k.

    python tools/merge_microbench.py [--blocks 16777216] [--n 32] [--reps 20]

Random PDM bytes (the merge is data-independent), L2 flushed before every
timed launch, CUDA events on the launching stream.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
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
    ap.add_argument("--ks", type=int, nargs="+", default=[1, 2, 4, 8, 16, 24, 32])
    ap.add_argument("--no-host", action="store_true", help="skip the D' to host section")
    ap.add_argument("--packed", action="store_true",
                    help="also time pdm_combine_packed (planes are random walks along z, "
                         "so they pack)")
    args = ap.parse_args()
    L = _lib.lib()
    nb, n = args.blocks, args.n
    pitch = device.plane_pitch(nb) + int(os.environ.get("PDM_MB_RAW_PAD", "0"))
    if args.packed:  # 1-Lipschitz rows of 256 blocks, like distance fields
        steps = torch.randint(-1, 2, (n, pitch // 256, 256), dtype=torch.int16, device="cuda")
        start = torch.randint(0, 256, (n, pitch // 256, 1), dtype=torch.int16, device="cuda")
        walk = (start + steps.cumsum(2)).clamp_(0, 255)
        pdms = walk.to(torch.uint8).reshape(n, pitch).contiguous()
        del steps, start, walk
    else:
        pdms = torch.randint(0, 256, (n, pitch), dtype=torch.uint8, device="cuda")
    out = torch.empty(nb, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    drain = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")

    class _Flush:  # write 256 MB, then read 256 MB (dirty lines drained untimed)
        @staticmethod
        def fill_(v):
            flush.fill_(v)
            drain.sum()
    st = _lib.stream_handle()
    res = {}
    for k in args.ks:
        if k > n:
            break
        sel = np.ascontiguousarray(np.arange(k), dtype=np.int32)
        ts = []
        for r in range(args.reps + 3):
            _Flush.fill_(r & 0xFF)
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
    packed = {}
    if args.packed:
        chunks = int(L.pdm_packed_chunks(nb))
        nib_pitch, base_pitch = -(-chunks * 8 // 256) * 256, -(-chunks // 256) * 256
        nib_pitch += int(os.environ.get("PDM_MB_NIB_PAD", "0"))  # plane-stride experiments
        base_pitch += int(os.environ.get("PDM_MB_BASE_PAD", "0"))
        nib = torch.empty((n, nib_pitch), dtype=torch.uint8, device="cuda")
        base = torch.empty((n, base_pitch), dtype=torch.uint8, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(L.pdm_pack_pdms(_lib.ptr(pdms), pitch, nb, n, _lib.ptr(nib), nib_pitch,
                                   _lib.ptr(base), base_pitch, _lib.ptr(bad), st), "pack")
        assert int(bad.item()) == 0
        for k in args.ks:
            if k > n:
                break
            sel = np.ascontiguousarray(np.arange(k), dtype=np.int32)
            ts = []
            for r in range(args.reps + 3):
                _Flush.fill_(r & 0xFF)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(L.pdm_combine_packed(_lib.ptr(nib), nib_pitch, _lib.ptr(base),
                                                base_pitch, None, nb, n, sel.ctypes.data, k,
                                                _lib.ptr(out), None, st), "pdm_combine_packed")
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            moved = k * nb * 9 / 16 + nb
            packed[k] = {"ms": round(ms, 5), "moved GB/s": round(moved / (ms * 1e-3) / 1e9, 1),
                         "effective GB/s": round((k + 1) * nb / (ms * 1e-3) / 1e9, 1)}
            if not os.environ.get("PDM_MB_NOCHECK"):
                assert torch.equal(out, pdms[:k, :nb].min(dim=0).values)
    # floor for the same bytes as k=1: a plain device copy of one map
    ts = []
    for r in range(args.reps + 3):
        _Flush.fill_(r & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out.copy_(pdms[1, :nb])
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    res["torch_copy_1map"] = {"ms": round(ms, 5), "GB/s": round(2 * nb / (ms * 1e-3) / 1e9, 1)}
    # D' to host: merge into HBM + D2H copy, vs the merge writing pinned host
    # memory directly (zero-copy over PCIe)
    to_host = {}
    host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    for k in (() if args.no_host else (1, 16, 32)):
        sel = np.ascontiguousarray(np.arange(k), dtype=np.int32)
        modes = ("hbm+d2h", "zero-copy") + (("packed hbm+d2h", "packed zero-copy",
                                              "packed->packed zero-copy")
                                             if args.packed else ())
        for mode in modes:
            ts = []
            for r in range(8):
                _Flush.fill_(r & 0xFF)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dst = out if mode.endswith("hbm+d2h") else host
                if mode == "packed->packed zero-copy":  # D' itself packed (9/16 of the bytes)
                    _lib.check(L.pdm_combine_packed_to_packed(
                        _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, nb, n,
                        sel.ctypes.data, k, _lib.ptr(host), _lib.ptr(host) + chunks * 8, st),
                        "pdm_combine_packed_to_packed")
                elif mode.startswith("packed"):
                    _lib.check(L.pdm_combine_packed(_lib.ptr(nib), nib_pitch, _lib.ptr(base),
                                                    base_pitch, None, nb, n, sel.ctypes.data, k,
                                                    _lib.ptr(dst), None, st), "pdm_combine_packed")
                else:
                    _lib.check(L.pdm_combine(_lib.ptr(pdms), pitch, nb, n, sel.ctypes.data, k,
                                             _lib.ptr(dst), st), "pdm_combine")
                if mode.endswith("hbm+d2h"):
                    host.copy_(out, non_blocking=True)
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            moved = chunks * 9 if mode == "packed->packed zero-copy" else nb
            to_host[f"{mode} k={k}"] = {"ms": round(ms, 4), "PCIe GB/s": round(moved / ms / 1e6, 1)}
            if mode != "packed->packed zero-copy":
                assert torch.equal(host.cuda(), pdms[:k, :nb].min(dim=0).values)
    print(json.dumps({"blocks": nb, "n": n, "merge": res, "packed": packed, "to_host": to_host}))


if __name__ == "__main__":
    main()
