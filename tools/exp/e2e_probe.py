"""Where the public-API TF-change step spends its time (config c and 256^3):
select_partitions (alpha gather, H2D, select kernel, sync), combine (merge +
sync), .dist (D' encode -> PCIe -> host expand).  Wall-clock medians, L2
flushed before each rep.  Also: per-step times of two back-to-back timed
passes of the bench loop (first-step anomaly)."""
import json, os, sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import torch
    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import _lib, synth, device
    from paper_2407_21552_b200.transfer import _AlphaStage
    L = _lib.lib()
    res = {"omp_env": {k: v for k, v in os.environ.items() if k.startswith("OMP") or k.startswith("GOMP")}}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn, reps=30, pre=None):
        ts = []
        for r in range(reps + 3):
            flush.fill_(r & 0xFF)
            if pre:
                pre(r)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append((time.perf_counter() - t0) * 1e3)
        return round(float(np.median(ts)), 4)

    for dims, b, n in (((1024,) * 3, 4, 32), ((256,) * 3, 4, 64)):
        vol = synth.synth_volume_device(dims, 16, seed=2407, nbox=12)
        grid = pdm.BlockGrid.for_dims(dims, b)
        scheme = pdm.scheme_uniform(n, 16)
        pset = pdm.build_pdm_set(vol, grid, scheme)
        rng = np.random.default_rng(1)
        luts = []
        for i in range(40):
            lut = np.zeros((65536, 4))
            picks = rng.choice(n, n // 2, replace=False)
            for p in picks:
                part = scheme.partitions[p]
                lut[part.rho_lo:part.rho_hi + 1, 3] = 0.5
            luts.append(lut)
        tfs = [pdm.TransferFunction(lut=l) for l in luts]
        r = {}
        dst = torch.empty(65536, dtype=torch.float64, pin_memory=True)
        it = iter(range(10 ** 9))
        r["gather_cold_luts"] = timed(lambda: L.pdm_gather_f64_host(
            luts[next(it) % 40].ctypes.data + 24, 65536, 4, dst.data_ptr()))
        r["gather_same_lut"] = timed(lambda: L.pdm_gather_f64_host(
            luts[0].ctypes.data + 24, 65536, 4, dst.data_ptr()))
        r["np_copy_column"] = timed(lambda: np.copyto(dst.numpy(), luts[0][:, 3]))
        stage = scheme._alpha_stage(_lib.stream_handle())
        r["upload_into"] = timed(lambda: _AlphaStage.upload_into(tfs[0], stage))
        r["select_partitions"] = timed(lambda: pdm.select_partitions(tfs[next(it) % 40], scheme))
        sel = pdm.select_partitions(tfs[0], scheme)
        r["combine"] = timed(lambda: pdm.combine(pset, sel))
        hold = {}
        r["dist"] = timed(lambda: hold["dm"].dist,
                          pre=lambda i: hold.__setitem__("dm", pdm.combine(pset, sel)))
        r["step_total"] = timed(lambda: pdm.combine(pset, pdm.select_partitions(
            tfs[next(it) % 40], scheme)).dist)
        dm = pdm.combine(pset, sel)
        out = device.host_buffer(grid.bdims)
        stage_n, stage_b = pset._host_stage()
        nb = grid.num_blocks
        for pieces in (1, 2, 4):
            r[f"dprime_to_host_p{pieces}"] = timed(lambda: L.pdm_dprime_to_host(
                _lib.ptr(dm.device()), nb, _lib.ptr(stage_n), _lib.ptr(stage_b), out.ctypes.data,
                pieces, 3, _lib.stream_handle()))
        r["unpack_sparse_only"] = timed(lambda: L.pdm_unpack_sparse_host(
            _lib.ptr(stage_n), nb, out.ctypes.data))
        flags = pdm.select_partitions_device(pdm.transfer.alpha_to_device(tfs[0]), scheme)
        r["merge_packed_to_host_old"] = timed(lambda: pdm.acceleration._host_packed_pays(pset) and
            L.pdm_merge_packed_to_host(*_old_args(pset, flags, out, L)))
        sel_idx = np.ascontiguousarray([i - 1 for i in sel.sorted], dtype=np.int32)
        nib, nib_pitch, base, base_pitch = pset.packed()
        dprime = device.empty(grid.bdims, np.uint8)
        pieces = max(1, min(16, (-(-nb // 32)) // pdm.acceleration._HOST_PIECE_ITEMS))
        r["combine_dual_c"] = timed(lambda: L.pdm_combine_packed_host(
            _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, pset.tile_bounds_ptr(), nb, pset.n, None,
            sel_idx.ctypes.data, int(sel_idx.size), _lib.ptr(dprime), _lib.ptr(stage_n),
            out.ctypes.data, pieces, _lib.stream_handle()))
        r["merge_to_host_idx_c"] = timed(lambda: L.pdm_merge_packed_to_host(
            _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, pset.tile_bounds_ptr(), nb, pset.n, None,
            sel_idx.ctypes.data, int(sel_idx.size), _lib.ptr(stage_n), _lib.ptr(stage_b),
            out.ctypes.data, pieces, 3, _lib.stream_handle()))

        def reader_combine():
            pset._last_probe = pdm.acceleration._HostReadProbe()
            pset._last_probe.read = True
            return pdm.combine(pset, sel).dist

        r["combine_dual_py_dist"] = timed(reader_combine)
        r["step_total_reader"] = timed(lambda: pdm.combine(pset, pdm.select_partitions(
            tfs[next(it) % 40], scheme)).dist)
        res[f"{dims[0]}^3_n{n}"] = r
        del pset, vol
    print(json.dumps(res, indent=1))


def _old_args(pset, flags, out, L):
    from paper_2407_21552_b200 import _lib
    nib, nib_pitch, base, base_pitch = pset.packed()
    nib_h, base_h = pset._host_stage()
    return (_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch, None, pset.grid.num_blocks, pset.n,
            _lib.ptr(flags), None, 0, _lib.ptr(nib_h), _lib.ptr(base_h), out.ctypes.data, 2, 3,
            _lib.stream_handle())


if __name__ == "__main__":
    main()
