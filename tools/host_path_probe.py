"""Where the time of combine(...).dist goes at config c (packed D' to host):
kernel-only zero-copy, host expansion alone, and the one-call pipeline with
1/2/4/8 pieces.  Wall-clock medians over 30 runs, L2 flushed before each."""
import json, sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import _lib, synth
    L = _lib.lib()
    vol = synth.synth_volume_device((1024, 1024, 1024), 16, seed=2407, nbox=12)
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    scheme = pdm.scheme_uniform(32, 16)
    pset = pdm.build_pdm_set(vol, grid, scheme)
    nib, nib_pitch, base, base_pitch = pset.packed()
    nib_h, base_h = pset._host_stage()
    nb = grid.num_blocks
    chunks = int(L.pdm_packed_chunks(nb))
    sel = np.ascontiguousarray(np.arange(0, 32, 2), dtype=np.int32)  # k = 16
    from paper_2407_21552_b200 import device
    out = device.host_buffer((nb,))  # 64-byte aligned, as .dist gets
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = _lib.stream_handle()

    def timed(fn, reps=30):
        ts = []
        for r in range(reps + 3):
            flush.fill_(r & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append((time.perf_counter() - t0) * 1e3)
        return round(float(np.median(ts)), 4)

    res = {}
    res["kernel_zero_copy"] = timed(lambda: L.pdm_combine_packed_to_packed(
        _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, nb, 32, sel.ctypes.data, 16,
        _lib.ptr(nib_h), _lib.ptr(base_h), st))
    res["unpack_only"] = timed(lambda: L.pdm_unpack_packed_host(
        _lib.ptr(nib_h), _lib.ptr(base_h), nb, out.ctypes.data))
    res["unpack_delta_only"] = timed(lambda: L.pdm_unpack_delta_host(
        _lib.ptr(nib_h), _lib.ptr(base_h), nb, out.ctypes.data))
    for pieces in (1, 2, 4, 8, 16):  # 3 = sparse delta D' (the default)
        res[f"pipeline_f3_{pieces}"] = timed(lambda: L.pdm_merge_packed_to_host(
            _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, None, nb, 32, None,
            sel.ctypes.data, 16, _lib.ptr(nib_h), _lib.ptr(base_h), out.ctypes.data,
            pieces, 3, st))
    res["unpack_sparse_only"] = timed(lambda: L.pdm_unpack_sparse_host(
        _lib.ptr(nib_h), nb, out.ctypes.data))
    for fmt in (1, 2):  # 1 = nibble D', 2 = 2-bit delta D'
        for pieces in (1, 2, 4, 8):
            res[f"pipeline_f{fmt}_{pieces}"] = timed(lambda: L.pdm_merge_packed_to_host(
                _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, None, nb, 32, None,
                sel.ctypes.data, 16, _lib.ptr(nib_h), _lib.ptr(base_h), out.ctypes.data,
                pieces, fmt, st))
    s = pdm.PartitionSelection(selected=frozenset(int(i) + 1 for i in sel), n=32)
    res["api_dist"] = timed(lambda: pdm.combine(pset, s).dist)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
