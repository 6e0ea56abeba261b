"""Distance-map update bench (BASELINE.json metric: "distance-map update ms per
TF change & Gvoxel/s vs HBM roofline, 1/2/4/8 B200").

One step = one transfer-function change: selection (K8) + min-merge over the
selected partitions' distance maps (K7) for BASELINE config c -- a 1024^3
uint16 volume, b=4 (256^3 blocks), n=32 partitions -- cycling through aligned
TFs selecting k = 1..32 partitions (the config's sweep).  Multi-GPU is weak
scaling: each rank owns one 1024-plane x-slab of a (1024*N, 1024, 1024)
volume and its slab of every PDM; the update needs no collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line on rank 0.  `value` = Gvoxel/s of the device-resident
update (alpha already in HBM, inputs > L2 and L2 flushed between steps);
`e2e` = the same metric through the public API (select_partitions + combine
+ DistanceMap.dist) with the TF read from and D' written to host memory.
`--impl reference` times the CPU oracle (the reference algorithm restated in
C, oracle/, all host threads) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG = {"dims": (1024, 1024, 1024), "bits": 16, "b": 4, "n": 32, "mode": "range_apron",
       "seed": 2407, "nbox": 12}
WORKLOAD = ("c: 1024^3 uint16 volume, 4^3 blocks (256^3), 32 partitions, TF changes "
            "selecting k=1..32 partitions (cycled)")
FLUSH_BYTES = 256 << 20


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


HOST_FORMATS = {
    0: "uint8 D'",
    1: "packed D' (base + 4-bit offsets per 16 blocks), expanded on the host",
    2: "packed D' (base + 2-bit z-deltas per 16 blocks), expanded on the host",
    3: "sparse packed D' (per 16 blocks: nothing if all zero, the base if flat, else base "
       "+ 2-bit z-deltas; 16 B of chunk bitmaps per 64 chunks), expanded on the host",
}


def d2h_bytes_per_step(pset, fmt: int, alphas, out) -> int:
    """Mean bytes the e2e step's D' moves over PCIe (untimed recount): fixed
    for formats 0-2; for the sparse form, 16 bitmap bytes per 64 chunks plus
    a base per non-zero chunk and a 4-byte code per non-flat chunk, counted
    from each step's D' (recomputed on the device)."""
    import torch

    import paper_2407_21552_b200 as pdm

    B = pset.grid.num_blocks
    items = -(-B // 32)
    if fmt == 0:
        return B
    if fmt in (1, 2):
        return items * (18 if fmt == 1 else 10)
    total = 0
    for a in alphas:
        pdm.update_from_tf(pset, torch.as_tensor(a, device=out.device), out=out)
        flat = out.reshape(-1)
        pad = (-flat.numel()) % 16
        if pad:
            flat = torch.cat([flat, flat[-1:].expand(pad)])
        ch = flat.view(-1, 16)
        mn, mx = ch.amin(1), ch.amax(1)
        is_flat = mn == mx
        nonzero = ~(is_flat & (mn == 0))
        total += 16 * -(-items // 32) + int(nonzero.sum()) + 4 * int((~is_flat).sum())
    return round(total / len(alphas))


def tf_sequence(n: int, span: int, steps: int, seed: int):
    """Aligned TFs (support = union of k whole partitions), k = 1..n cycled."""
    from paper_2407_21552_b200 import scheme_uniform

    scheme = scheme_uniform(n, int(np.log2(span)))
    rng = np.random.default_rng(seed)
    out = []
    for i in range(steps):
        k = (i % n) + 1
        picks = rng.choice(np.arange(n), size=k, replace=False)
        alpha = np.zeros(span)
        for p in picks:
            lo, hi = scheme.partitions[p].rho_lo, scheme.partitions[p].rho_hi
            alpha[lo: hi + 1] = rng.uniform(0.05, 1.0, hi - lo + 1)
        out.append((k, alpha))
    return out


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every
    ~2 ms from a background thread while the timed region runs (the same
    counters `nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.*` reads)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            idx = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(self.gpu)).split(",")[self.gpu]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES", "").replace(",", "").isdigit() else self.gpu
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception as exc:  # no NVML: report unsampled
            self._err = str(exc)
            self._nvml = None
        return self

    def _run(self):
        p = self._nvml
        while not self._stop.is_set():
            try:
                sm = p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)
                rs = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        reasons = sorted({name for _, rs in self.samples for bit, name in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML clocks + clocks_event_reasons, 2 ms polling"}


# ---------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------

def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import sharded, synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    nx, ny, nz = CFG["dims"]
    bits, b, n = CFG["bits"], CFG["b"], CFG["n"]
    span = 1 << bits
    gdims = (nx * world, ny, nz)
    x0, x1 = rank * nx, (rank + 1) * nx

    # ---- setup (untimed): device-born volume slab, PDM precompute ----------------
    vol = synth.synth_volume_device(gdims, bits, seed=CFG["seed"], nbox=CFG["nbox"],
                                    x_range=(x0, x1))
    scheme = pdm.scheme_uniform(n, bits)
    grid = pdm.BlockGrid.for_dims(vol.dims, b)
    def precompute():
        if world > 1:
            return sharded.build_pdm_set_sharded(vol, b, scheme, CFG["mode"], x0 // b)
        return pdm.build_pdm_set(vol, grid, scheme, CFG["mode"])

    build_ms = []
    pset = None
    for _ in range(2):  # first call pays one-time costs (kernel attributes, allocations)
        pset = None  # release the previous set so the second build reuses its memory
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pset = precompute()
        torch.cuda.synchronize()
        build_ms.append((time.perf_counter() - t0) * 1e3)
    precompute_ms = build_ms[1]
    B = grid.num_blocks
    voxels_rank = vol.num_voxels

    steps, warm = args.steps, args.warmup
    seq = tf_sequence(n, span, warm + steps, CFG["seed"] + 1)
    alphas = [torch.from_numpy(a).to(dev) for _, a in seq]
    out = torch.empty(grid.bdims, dtype=torch.uint8, device=dev)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    flush_w = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    flush_r = torch.zeros(FLUSH_BYTES // 8, dtype=torch.int64, device=dev)

    def flush_l2(i):
        """Untimed L2 flush between steps: write 256 MB (> 126 MB L2), then read
        another 256 MB so the dirty lines are written back now rather than
        inside the next timed step."""
        flush_w.fill_(i & 0xFF)
        flush_r.sum()

    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident update (value) --------------------------------------------
    for i in range(warm):
        pdm.update_from_tf(pset, alphas[i], out=out, flags=flags)
    def timed_pass(merge_only):
        """One timed pass over the K steps; events bracket each step only (an
        event between select and merge would defeat the PDL overlap).  With
        merge_only the flags are selected untimed first and the events bracket
        the merge kernel alone (the roofline's per-launch duration)."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        if args.gpu_lead_ms > 0:
            # keep the GPU busy while the host enqueues, so no step waits on a launch
            torch.cuda._sleep(int(args.gpu_lead_ms * 1e-3 * 1.9e9))
        for i in range(steps):
            flush_l2(i)  # evict the previous step's maps from L2 (untimed)
            if merge_only:
                pdm.select_partitions_device(alphas[warm + i], scheme, flags)
            ev[i][0].record(stream)
            if not merge_only:
                pdm.select_partitions_device(alphas[warm + i], scheme, flags)
            pdm.acceleration.combine_flags_into(pset, flags, out)
            ev[i][1].record(stream)
        barrier()
        return [a.elapsed_time(b) for a, b in ev]

    barrier()
    with ClockSampler(local_rank) as clocks:
        time.sleep(0.02)  # sampler running before the first timed step
        step_ms = timed_pass(merge_only=False)
    merge_ms = timed_pass(merge_only=True)
    ks = [k for k, _ in seq[warm:warm + steps]]
    total_ms = sum(step_ms)
    merge_bytes = sum((k + 1) * B for k in ks)  # SURVEY.md §8(d) algorithmic bytes
    packed = pset.packed()
    # D' form the e2e step ships to the host (acceleration._packed_to_host)
    host_packed = pdm.acceleration._host_packed_pays(pset)
    host_fmt = pdm.acceleration._host_format(pset) if host_packed else 0
    if packed is not None:  # bytes the packed merge actually moves: nibbles + bases + D'
        per_plane = -(-B // 32) * 2 * 9
        moved_bytes = sum(k * per_plane + B for k in ks)
    else:
        moved_bytes = merge_bytes

    # parity spot check of the last step against the host-API path (untimed)
    last = pdm.PartitionSelection(
        selected=frozenset(int(i) + 1 for i in np.flatnonzero(flags.cpu().numpy())), n=n)
    assert torch.equal(pdm.combine(pset, last).device(), out), "fused vs API mismatch"

    # ---- end-to-end through the public API with host buffers -------------------------
    host_tfs = []
    for _, a in seq[warm:warm + steps]:
        lut = np.zeros((span, 4))
        lut[:, 3] = a
        host_tfs.append(pdm.TransferFunction(lut=lut))
    for i in range(min(warm, steps)):
        pdm.combine(pset, pdm.select_partitions(host_tfs[i], scheme)).dist
    e2e_s = 0.0
    parts = np.zeros(3)  # select_partitions / combine (launch) / .dist (merge + D2H)
    barrier()
    for i in range(steps):
        flush_l2(i)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sel = pdm.select_partitions(host_tfs[i], scheme)
        t2 = time.perf_counter()
        dm = pdm.combine(pset, sel)
        t3 = time.perf_counter()
        host = dm.dist  # D2H into pinned host memory
        t4 = time.perf_counter()
        e2e_s += t4 - t1
        parts += (t2 - t1, t3 - t2, t4 - t3)
    assert host.shape == grid.bdims
    e2e_parts_ms = (parts / steps * 1e3).round(4).tolist()
    barrier()
    d2h_bytes = d2h_bytes_per_step(pset, host_fmt, [a for _, a in seq[warm:warm + steps]], out)

    # ---- max over ranks ----------------------------------------------------------------
    vals = torch.tensor([total_ms, e2e_s * 1e3, sum(merge_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, merge_total_ms = vals.tolist()
    clock = clocks.summary()
    if rank != 0:
        return None

    gvox = voxels_rank * world * steps / (total_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    achieved = merge_bytes / (merge_total_ms * 1e-3) / 1e9
    line = {
        "metric": "distance-map update Gvoxel/s per TF change (select + merge), HBM roofline",
        "value": round(gvox, 2),
        "unit": "Gvoxel/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": round(total_ms / steps, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (device-born hash-box volume, seeded; aligned TFs)",
        "config": {"workload": WORKLOAD, "dims_per_gpu": list(CFG["dims"]),
                   "global_dims": list(gdims), "bits": bits, "b": b, "n": n,
                   "occupancy_mode": CFG["mode"], "k_sweep": "1..32",
                   "l2": "inputs > L2 (PDM set 537 MB/GPU); untimed L2 flush between steps "
                         "(256 MB write, then 256 MB read to drain dirty lines)",
                   "parallelism": f"x-slab x{world}, no collective on the update"},
        "roofline": {"bound": "hbm",
                     "kernel": ("combine_packed_flags_kernel (K7 merge over nibble-packed planes)"
                                if packed is not None else "combine_flags_kernel (K7 merge)"),
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "algorithmic_bytes": "(k+1) * num_blocks per launch (SURVEY.md 8(d))",
                     "moved_bytes_per_step": round(moved_bytes / steps),
                     "moved_GBps": round(moved_bytes / (merge_total_ms * 1e-3) / 1e9, 1),
                     "moved_frac": round(moved_bytes / (merge_total_ms * 1e-3) / 1e9 / peak, 4),
                     "traffic": traffic_from_profiles(), "merge_ms_per_step":
                         round(merge_total_ms / steps, 5)},
        "e2e": {"value": round(voxels_rank * world * steps / (e2e_ms * 1e-3) / 1e9, 2),
                "unit": "Gvoxel/s", "ms_per_step": round(e2e_ms / steps, 4),
                "h2d_bytes_per_step": span * 8,
                "d2h_bytes_per_step": d2h_bytes,
                "d2h_format": HOST_FORMATS[host_fmt],
                "api": "select_partitions(tf, scheme) + combine(pdm_set, sel) + .dist",
                "breakdown_ms": {"select_partitions": e2e_parts_ms[0], "combine_launch": e2e_parts_ms[1], "dist_merge_d2h": e2e_parts_ms[2]}},
        "gpu_launches": 2 * steps,
        "clocks": clock,
        "precompute_ms": round(precompute_ms, 2),
        "precompute_first_call_ms": round(build_ms[0], 2),
        "sweep_ms": {str(k): round(t, 5) for k, t in sorted(zip(ks, step_ms))[:: max(1, steps // 8)]},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(pset, seq[warm:warm + steps], scheme)
    return line


def traffic_from_profiles():
    p = ROOT / "profiles" / "merge_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get("traffic_bytes_per_launch")


def cpu_baseline_sample(pset, seq, scheme):
    """The CPU oracle (reference algorithm in C, all host threads) on the same
    PDM bytes: select + combine for the same TF sequence (bounded sample)."""
    import oracle

    threads = oracle.max_threads()
    oracle.set_threads(threads)
    nb = pset.grid.num_blocks
    maps = pset.storage[:, :nb].cpu().numpy()
    bounds = scheme.bounds()
    out = np.empty(nb, dtype=np.uint8)
    budget_s, done, t_total = 15.0, 0, 0.0
    for k, alpha in seq:
        t0 = time.perf_counter()
        sel = oracle.select(alpha, bounds)
        oracle.combine(maps, sel, out=out)
        t_total += time.perf_counter() - t0
        done += 1
        if t_total > budget_s:
            break
    vox = pset.grid.num_blocks * pset.grid.b ** 3
    return {"value": round(vox * done / t_total / 1e9, 3), "unit": "Gvoxel/s", "cores": threads,
            "kind": "port", "ms_per_step": round(t_total / done * 1e3, 3),
            "sample": f"{done} TF changes of the timed sequence (k cycled), oracle select+combine "
                      f"on the GPU-built PDM set copied to host"}


# ---------------------------------------------------------------------------------
# reference arm: the CPU oracle (reference algorithm restated in C) on host cores
# ---------------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle
    from paper_2407_21552_b200.synth import synth_boxes

    oracle.build()
    threads = oracle.max_threads()
    oracle.set_threads(threads)
    nx, ny, nz = CFG["dims"]
    bits, b, n = CFG["bits"], CFG["b"], CFG["n"]
    span = 1 << bits
    gdims = (nx * world, ny, nz)
    boxes = synth_boxes(gdims, bits, CFG["seed"], CFG["nbox"])
    t0 = time.perf_counter()
    vox = oracle.synth_volume(bits, gdims, boxes, CFG["seed"], x_range=(0, nx))
    bounds = [(i * (span // n), (i + 1) * (span // n) - 1) for i in range(n)]
    pdms = oracle.build_pdm_set(vox, b, bounds, CFG["mode"])
    setup_s = time.perf_counter() - t0
    del vox
    steps, warm = args.steps, args.warmup
    seq = tf_sequence(n, span, warm + steps, CFG["seed"] + 1)
    out = np.empty(pdms.shape[1:], dtype=np.uint8)
    for _, a in seq[:warm]:
        oracle.combine(pdms, oracle.select(a, bounds), out=out)
    times = []
    for _, a in seq[warm:warm + steps]:
        t1 = time.perf_counter()
        oracle.combine(pdms, oracle.select(a, bounds), out=out)
        times.append(time.perf_counter() - t1)
    total = sum(times)
    voxels = nx * ny * nz
    val = voxels * steps / total / 1e9
    return {
        "metric": "distance-map update Gvoxel/s per TF change (select + merge), HBM roofline",
        "impl": "reference",
        "value": round(val, 3),
        "unit": "Gvoxel/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": round(total / steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (same hash-box volume slab and TF sequence as the b200 arm)",
        "config": {"workload": WORKLOAD, "dims_per_gpu": list(CFG["dims"]), "bits": bits,
                   "b": b, "n": n, "occupancy_mode": CFG["mode"], "k_sweep": "1..32"},
        "cpu_baseline": {"value": round(val, 3), "unit": "Gvoxel/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{steps} TF changes (select + combine) on the full config-c "
                                   f"PDM set; setup (volume + PDM build) {setup_s:.1f}s untimed"},
        "e2e": {"value": round(val, 3), "unit": "Gvoxel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gpu-lead-ms", type=float, default=0.0,
                    help="GPU spin before each timed pass so host enqueue never gates a step")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "b200":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_b200(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and args.impl == "b200":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
