"""Distance-map update bench (BASELINE.json metric: "distance-map update ms per
TF change & Gvoxel/s vs HBM roofline, 1/2/4/8 B200").

One step = one transfer-function change: selection (K8) + min-merge over the
selected partitions' distance maps (K7).  Workloads (BASELINE.json configs):

  --config c (default)  1024^3 uint16 volume, b=4 (256^3 blocks), n=32
                        range_apron PDMs.  Multi-GPU is weak scaling: rank r
                        owns x-slab r of a (1024*N, 1024, 1024) volume and its
                        slab of every PDM; the update needs no collective.
  --config d            2048^3 uint16, b=4, n=32, split into N x-slabs
                        (strong scaling): the sharded precompute (boundary
                        voxel planes + DT edge all_gather over NCCL) is timed
                        too, then the same update sweep on every rank's slab.

The timed TF changes select k = 1..n partitions (aligned TFs): every k once
when --steps >= n, else k spaced evenly over 1..n (mean k = (n+1)/2 either
way); warm-up uses separate TFs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c|d]
                  [--impl b200|reference] [--no-parity] [--no-cpu-baseline]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks.  Prints ONE JSON line on rank 0.
`value` = Gvoxel/s of the device-resident update (alpha already in HBM, inputs
> L2 and L2 flushed between steps); `e2e` = the same metric through the
public API (select_partitions + combine + DistanceMap.dist) with the TF read
from and D' written to host memory.  `parity` = every timed D' (and, at N=1,
every PDM plane) compared with the CPU oracle built from the same volume
bytes; a mismatch exits non-zero.  `--impl reference` times the CPU oracle
(the reference algorithm restated in C, oracle/, all host threads) on the
same workload and, beside it, the shipped reference package (numba/numpy,
baseline/_ref) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "distance-map update Gvoxel/s per TF change (select + merge), HBM roofline"
CONFIGS = {
    "c": {"dims": (1024, 1024, 1024), "bits": 16, "b": 4, "n": 32, "mode": "range_apron",
          "seed": 2407, "nbox": 12, "scaling": "weak",
          "workload": "c: 1024^3 uint16 volume, 4^3 blocks (256^3), 32 partitions, TF changes "
                      "selecting k=1..32 partitions"},
    "d": {"dims": (2048, 2048, 2048), "bits": 16, "b": 4, "n": 32, "mode": "range_apron",
          "seed": 2407, "nbox": 12, "scaling": "strong",
          "workload": "d: 2048^3 uint16 volume, 4^3 blocks (512^3), 32 partitions, x-slab sharded "
                      "over the GPUs (sharded precompute + TF changes selecting k=1..32)"},
}
FLUSH_BYTES = 256 << 20
DPRIME_BUDGET = 40 << 30  # device bytes for per-step D' buffers (parity of every timed step)
REF_SAMPLE_S = 15.0  # bounded CPU samples


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


def timed_ks(n: int, steps: int) -> list[int]:
    """k for each timed step: 1..n cycled when steps >= n, else evenly spaced
    over 1..n (both ends included)."""
    if steps >= n:
        return [(i % n) + 1 for i in range(steps)]
    if steps == 1:
        return [(n + 1) // 2]
    return [1 + round(i * (n - 1) / (steps - 1)) for i in range(steps)]


def aligned_alpha(scheme, picks, rng) -> np.ndarray:
    alpha = np.zeros(scheme.intensity_span)
    for p in picks:
        part = scheme.partitions[p - 1]
        alpha[part.rho_lo: part.rho_hi + 1] = rng.uniform(0.05, 1.0, part.width)
    return alpha


def tf_plan(n: int, bits: int, steps: int, warm: int, seed: int):
    """(warm-up TFs, timed TFs): lists of (picks 1-based sorted, alpha)."""
    from paper_2407_21552_b200 import scheme_uniform

    scheme = scheme_uniform(n, bits)
    rng = np.random.default_rng(seed)

    def one(k):
        picks = sorted(int(p) for p in rng.choice(np.arange(1, n + 1), size=k, replace=False))
        return picks, aligned_alpha(scheme, picks, rng)

    warm_tfs = [one(int(rng.integers(1, n + 1))) for _ in range(warm)]
    return warm_tfs, [one(k) for k in timed_ks(n, steps)]


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
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.gpu]) if vis.replace(",", "").isdigit() else self.gpu
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
            time.sleep(0.005)  # first sample lands before the timed region
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


def slab_of(cfg, rank, world):
    """(global dims, this rank's voxel x-range, block-plane start)."""
    from paper_2407_21552_b200 import sharded

    nx, ny, nz = cfg["dims"]
    if cfg["scaling"] == "weak":
        gdims = (nx * world, ny, nz)
        x0, x1 = rank * nx, (rank + 1) * nx
    else:
        gdims = (nx, ny, nz)
        xs = sharded.slab_bounds(nx, cfg["b"], world)
        x0, x1 = xs[rank], xs[rank + 1]
    return gdims, (x0, x1), x0 // cfg["b"]


def config_keys(cfg, gdims, world):
    return {"workload": cfg["workload"], "dims_per_gpu":
            [gdims[0] // world if cfg["scaling"] == "strong" else cfg["dims"][0],
             *cfg["dims"][1:]],
            "global_dims": list(gdims), "bits": cfg["bits"], "b": cfg["b"], "n": cfg["n"],
            "occupancy_mode": cfg["mode"], "k_sweep": f"1..{cfg['n']}",
            "l2": "inputs > L2 (PDM set >= 537 MB/GPU); untimed L2 flush between steps "
                  "(256 MB write, then 256 MB read to drain dirty lines)",
            "parallelism": f"x-slab x{world}, no collective on the update"}


def oracle_pdms(cfg, gdims, x_range):
    """The CPU oracle's PDM set for the rank's volume (same bytes as the GPU's)."""
    import oracle
    from paper_2407_21552_b200 import scheme_uniform
    from paper_2407_21552_b200.synth import synth_boxes

    oracle.build()
    oracle.set_threads(oracle.max_threads())
    bounds = scheme_uniform(cfg["n"], cfg["bits"]).bounds()
    boxes = synth_boxes(gdims, cfg["bits"], cfg["seed"], cfg["nbox"])
    assert x_range == (0, gdims[0]), "oracle parity covers the whole volume (N=1)"
    return oracle.build_pdm_set_synth(cfg["bits"], gdims, boxes, cfg["seed"], cfg["b"], bounds,
                                      cfg["mode"])


def merge_traffic(ks):
    """ncu dram bytes (read + write) per merge launch for the run's TF sequence,
    from profiles/merge_traffic.json -- per-k values measured by
    `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` over the same
    k = 1..32 sequence (tools/evidence.sh), averaged over this run's ks; a
    committed capture, not this run."""
    p = ROOT / "profiles" / "merge_traffic.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text())
    per_k = {int(k): v for k, v in (d.get("per_k") or {}).items()}
    if per_k and all(k in per_k for k in ks):
        return round(float(np.mean([per_k[k] for k in ks]))), d.get("source")
    pts = d.get("points") or [{"k": d["k"], "traffic_bytes_per_launch":
                              d["traffic_bytes_per_launch"]}]
    kk = np.array([q["k"] for q in pts], float)
    tr = np.array([q["traffic_bytes_per_launch"] for q in pts], float)
    mean_k = float(np.mean(ks))
    if len(pts) >= 2:
        slope, icpt = np.polyfit(kk, tr, 1)
        return round(float(icpt + slope * mean_k)), d.get("source")
    return round(float(tr[0] * (mean_k + 1) / (kk[0] + 1))), d.get("source")


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import sharded, synth

    cfg = CONFIGS[args.config]
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    bits, b, n = cfg["bits"], cfg["b"], cfg["n"]
    span = 1 << bits
    gdims, (x0, x1), bx0 = slab_of(cfg, rank, world)
    sharded_build = world > 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- setup (untimed): device-born volume slab, PDM precompute ----------------
    vol = synth.synth_volume_device(gdims, bits, seed=cfg["seed"], nbox=cfg["nbox"],
                                    x_range=(x0, x1))
    scheme = pdm.scheme_uniform(n, bits)
    grid = pdm.BlockGrid.for_dims(vol.dims, b)

    def precompute():
        if sharded_build:
            return sharded.build_pdm_set_sharded(vol, b, scheme, cfg["mode"], bx0)
        return pdm.build_pdm_set(vol, grid, scheme, cfg["mode"])

    build_ms = []
    pset = None
    for _ in range(2):  # first call pays one-time costs (kernel attributes, allocations)
        pset = None  # release the previous set so the second build reuses its memory
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pset = precompute()
        e1.record()
        barrier()
        build_ms.append(e0.elapsed_time(e1))
    B = grid.num_blocks
    voxels_rank = vol.num_voxels
    voxels_job = int(np.prod(gdims))
    del vol
    torch.cuda.empty_cache()

    # ---- parity inputs: the oracle's PDMs from the same bytes (N=1) ----------------
    check = not args.no_parity and world == 1
    want = None
    parity = {"checked": False}
    if check:
        t0 = time.perf_counter()
        want = oracle_pdms(cfg, gdims, (x0, x1))
        oracle_s = time.perf_counter() - t0
        bad_planes = [p for p in range(n) if not np.array_equal(
            pset.storage[p, :B].cpu().numpy(), want[p].reshape(-1))]
        parity = {"checked": True, "oracle_build_s": round(oracle_s, 1),
                  "pdm_planes": n, "pdm_planes_mismatched": len(bad_planes)}
        time.sleep(0.05)  # the oracle's OpenMP threads stop spinning before timing
    elif world > 1:
        parity = {"checked": False, "why": "N>1: the multi-rank build is checked against the "
                  "oracle by tests/test_sharded.py (gloo world 2/3; 2-rank GPU test)"}

    steps, warm = args.steps, args.warmup
    warm_tfs, timed_tfs = tf_plan(n, bits, steps, warm, cfg["seed"] + 1)
    ks = [len(p) for p, _ in timed_tfs]
    alphas_w = [torch.from_numpy(a).to(dev) for _, a in warm_tfs]
    alphas = [torch.from_numpy(a).to(dev) for _, a in timed_tfs]
    nbuf = max(1, min(steps, DPRIME_BUDGET // max(1, B)))
    outs = [torch.empty(grid.bdims, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
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
    for i in range(warm):  # (the flush's torch kernels load lazily: warm them too)
        flush_l2(i)
        pdm.update_from_tf(pset, alphas_w[i], out=outs[0], flags=flags)

    def timed_pass(merge_only):
        """One timed pass over the K steps; events bracket each step only (an
        event between select and merge would defeat the PDL overlap).  With
        merge_only the flags are selected untimed first and the events bracket
        the merge kernel alone (the roofline's per-launch duration).  An
        untimed warm step right before the loop keeps the GPU busy, so the
        first timed step does not start from an idle GPU."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        pdm.update_from_tf(pset, alphas_w[-1], out=outs[0], flags=flags)
        for i in range(steps):
            flush_l2(i)  # evict the previous step's maps from L2 (untimed)
            out = outs[i % nbuf]
            if merge_only:
                pdm.select_partitions_device(alphas[i], scheme, flags)
            ev[i][0].record(stream)
            if not merge_only:
                pdm.select_partitions_device(alphas[i], scheme, flags)
            pdm.acceleration.combine_flags_into(pset, flags, out)
            ev[i][1].record(stream)
        barrier()
        return [a.elapsed_time(b) for a, b in ev]

    barrier()
    with ClockSampler(local_rank) as clocks:
        step_ms = timed_pass(merge_only=False)
    if check:  # every timed D' whose buffer was not reused later
        bad = []
        for i in range(max(0, steps - nbuf), steps):
            import oracle

            wd = oracle.combine(want, timed_tfs[i][0])
            if not np.array_equal(outs[i % nbuf].cpu().numpy(), wd):
                bad.append(i)
        parity.update({"dprime_steps": min(steps, nbuf), "dprime_mismatched": len(bad)})
        time.sleep(0.05)  # the oracle's OpenMP threads stop spinning before the next pass
    # merge-only pass, counting the (1024-block tile, plane) pairs the packed
    # merges actually read (the per-tile skip drops planes that cannot lower a
    # tile): the moved bytes below are counted, not assumed
    L = pdm._lib.lib()
    pairs = torch.zeros(1, dtype=torch.int64, device=dev)
    L.pdm_merge_stats(pairs.data_ptr())
    try:
        merge_ms = timed_pass(merge_only=True)
    finally:
        L.pdm_merge_stats(None)
    pairs_read = int(pairs.item())
    total_ms = sum(step_ms)
    merge_bytes = sum((k + 1) * B for k in ks)  # SURVEY.md §8(d) algorithmic bytes
    packed = pset.packed()
    host_packed = pdm.acceleration._host_packed_pays(pset)
    host_fmt = pdm.acceleration._host_format(pset) if host_packed else 0
    tiles = -(-B // 1024)
    # selections of up to raw_k planes merge the raw planes (pdm_combine_flags_auto):
    # (k + 1) bytes per block; the others the packed planes with the tile skip
    raw_k = int(L.pdm_combine_raw_max_k()) if packed is not None else 0
    ks_raw = [k for k in ks if 1 <= k <= raw_k]
    ks_packed = [k for k in ks if k > raw_k]
    pairs_all = sum(ks_packed) * tiles
    if packed is not None:  # bytes the packed merge moves: nibbles + bases read, D' written
        moved_bytes = (pairs_read * 1024 * 9 // 16 + len(ks_packed) * B
                       + sum((k + 1) * B for k in ks_raw))
        if pset.tile_bounds_ptr() is not None:  # + the tile-bounds rows (2 B per pair)
            moved_bytes += 2 * pairs_all
    else:
        moved_bytes = merge_bytes

    # ---- end-to-end through the public API with host buffers -------------------------
    host_luts = []
    for _, a in timed_tfs:
        lut = np.zeros((span, 4))
        lut[:, 3] = a
        host_luts.append(lut)
    for picks, a in warm_tfs[:3]:
        lut = np.zeros((span, 4))
        lut[:, 3] = a
        tf = pdm.TransferFunction(lut=lut)
        pdm.combine(pset, pdm.select_partitions(tf, scheme)).dist
    e2e_bad = 0
    time.sleep(0.05)  # the oracle's OpenMP threads (parity check above) stop spinning
    if check:  # untimed parity pass over the same steps: every host D' vs the oracle
        import oracle

        for i in range(steps):
            tf = pdm.TransferFunction(lut=host_luts[i])
            host = pdm.combine(pset, pdm.select_partitions(tf, scheme)).dist
            e2e_bad += not np.array_equal(host, oracle.combine(want, timed_tfs[i][0]))
            del host
        parity.update({"e2e_host_steps": steps, "e2e_host_mismatched": e2e_bad})
        parity["ok"] = (parity["pdm_planes_mismatched"] == 0 and parity["dprime_mismatched"] == 0
                        and e2e_bad == 0)
        time.sleep(0.05)
        for picks, a in warm_tfs[:3]:  # back to the timed loop's steady state
            lut = np.zeros((span, 4))
            lut[:, 3] = a
            pdm.combine(pset, pdm.select_partitions(pdm.TransferFunction(lut=lut), scheme)).dist
    e2e_s = 0.0
    parts = np.zeros(3)  # select_partitions / combine (merge, completed) / .dist (D2H)
    barrier()
    for i in range(steps):  # timed pass: nothing but the API calls between the flushes
        tf = pdm.TransferFunction(lut=host_luts[i])  # the reference's TF (validated) -- untimed
        flush_l2(i)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sel = pdm.select_partitions(tf, scheme)
        t2 = time.perf_counter()
        dm = pdm.combine(pset, sel)
        t3 = time.perf_counter()
        host = dm.dist  # D' expanded into host memory
        t4 = time.perf_counter()
        e2e_s += t4 - t1
        parts += (t2 - t1, t3 - t2, t4 - t3)
        del dm, host
    e2e_parts_ms = (parts / steps * 1e3).round(4).tolist()
    barrier()
    d2h_bytes = d2h_bytes_per_step(pset, host_fmt, [a for _, a in timed_tfs], outs[0])

    # ---- max over ranks ----------------------------------------------------------------
    vals = torch.tensor([total_ms, e2e_s * 1e3, sum(merge_ms), build_ms[1]], dtype=torch.float64,
                        device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, merge_total_ms, build_max_ms = vals.tolist()
    clock = clocks.summary()
    if rank != 0:
        return None

    gvox = voxels_job * steps / (total_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    achieved = merge_bytes / (merge_total_ms * 1e-3) / 1e9
    mean_k = float(np.mean(ks))
    traffic, traffic_src = merge_traffic(ks)
    by, bz = grid.bdims[1], grid.bdims[2]
    line = {
        "metric": METRIC,
        "value": round(gvox, 2),
        "unit": "Gvoxel/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": round(total_ms / steps, 5),
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (device-born hash-box volume, seeded; aligned TFs)",
        "config": config_keys(cfg, gdims, world),
        "parity": parity,
        "roofline": {"bound": "hbm",
                     "kernel": ("combine_packed_flags_kernel (K7 merge over nibble-packed planes)"
                                if packed is not None else "combine_flags_kernel (K7 merge)"),
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "algorithmic_bytes": "(k+1) * num_blocks per launch (SURVEY.md 8(d)); "
                                          f"mean k {mean_k:.2f}",
                     "moved_bytes_per_step": round(moved_bytes / steps),
                     "planes_read_share": round(pairs_read / max(1, pairs_all), 4),
                     "moved_bytes_note": ("counted: (tile, plane) pairs the merge read x 576 B "
                                          "(nibbles + bases of 1024 blocks) + D' written + "
                                          "tile-bounds rows read"),
                     "moved_GBps": round(moved_bytes / (merge_total_ms * 1e-3) / 1e9, 1),
                     "moved_frac": round(moved_bytes / (merge_total_ms * 1e-3) / 1e9 / peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "merge_ms_per_step": round(merge_total_ms / steps, 5)},
        "e2e": {"value": round(voxels_job * steps / (e2e_ms * 1e-3) / 1e9, 2),
                "unit": "Gvoxel/s", "ms_per_step": round(e2e_ms / steps, 4),
                "h2d_bytes_per_step": span * 8,
                "d2h_bytes_per_step": d2h_bytes,
                "d2h_format": HOST_FORMATS[host_fmt],
                "api": "select_partitions(tf, scheme) + combine(pdm_set, sel) + .dist; each "
                       "call returns completed device work",
                "gpu_launches_per_step": 2 + (2 if host_fmt else 0),
                "breakdown_ms": {"select_partitions": e2e_parts_ms[0],
                                 "combine": e2e_parts_ms[1], "dist_d2h": e2e_parts_ms[2]}},
        "gpu_launches": 2 * steps,
        "clocks": clock,
        "precompute_ms": round(build_max_ms, 2),
        "precompute_first_call_ms": round(build_ms[0], 2),
        "precompute": ("sharded build_pdm_set (device-timed, max over ranks)" if sharded_build
                       else "build_pdm_set (device-timed)"),
        "sweep_ms": {str(k): round(t, 5) for k, t in sorted(zip(ks, step_ms))
                     [:: max(1, steps // 8)]},
    }
    if sharded_build:
        line["nccl_bytes_per_rank"] = {
            "apron_planes": 2 * 2 * gdims[1] * gdims[2] * (2 if bits == 16 else 1),
            "dt_edges_all_gather": world * 2 * n * by * bz}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(pset, want, timed_tfs, scheme, grid)
    if check and not parity["ok"]:
        print(json.dumps(line), flush=True)
        raise SystemExit("parity FAILED: GPU output differs from the CPU oracle")
    return line


def cpu_baseline_sample(pset, want, timed_tfs, scheme, grid):
    """The CPU oracle (reference algorithm in C, all host threads) on the same
    PDM bytes: select + combine for the timed TF sequence (bounded sample);
    beside it the shipped reference package (1 thread) when staged."""
    import oracle

    threads = oracle.max_threads()
    oracle.set_threads(threads)
    nb = grid.num_blocks
    maps = (want.reshape(want.shape[0], -1) if want is not None
            else pset.storage[:, :nb].cpu().numpy())
    bounds = scheme.bounds()
    out = np.empty(nb, dtype=np.uint8)
    done, t_total = 0, 0.0
    for _, alpha in timed_tfs:
        t0 = time.perf_counter()
        sel = oracle.select(alpha, bounds)
        oracle.combine(maps, sel, out=out)
        t_total += time.perf_counter() - t0
        done += 1
        if t_total > REF_SAMPLE_S:
            break
    vox = nb * grid.b ** 3
    res = {"value": round(vox * done / t_total / 1e9, 3), "unit": "Gvoxel/s", "cores": threads,
           "kind": "port", "ms_per_step": round(t_total / done * 1e3, 3),
           "sample": f"{done} TF changes of the timed sequence, oracle select+combine on the "
                     f"same PDM bytes"}
    shipped = shipped_reference_sample(maps.reshape((-1,) + grid.bdims), timed_tfs, scheme, grid)
    if shipped is not None:
        res["shipped_reference"] = shipped
    return res


def shipped_reference_sample(pdms, timed_tfs, scheme, grid):
    """The reference package as shipped (baseline/_ref: pdmrender, numpy +
    numba, single-threaded) timing its own select_partitions + combine on the
    same PDM bytes, wrapped in its own PdmSet (transfer.py:250-259,
    acceleration.py:244-276).  None when baseline/_ref is not staged."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "pdmrender").is_dir():
        return None
    sys.path.insert(0, str(ref_dir))
    try:
        import pdmrender as R
    except Exception as exc:  # staged but not importable here
        return {"unavailable": f"import failed: {exc}"}
    finally:
        sys.path.remove(str(ref_dir))
    rgrid = R.BlockGrid.for_dims(grid.dims, grid.b)
    rscheme = R.PartitionScheme(tuple(R.Partition(lo, hi) for lo, hi in scheme.bounds()))
    rset = R.PdmSet(grid=rgrid, scheme=rscheme, pdms=tuple(
        R.DistanceMap(b=grid.b, bdims=rgrid.bdims, dist=pdms[p]) for p in range(pdms.shape[0])),
        occupancy_mode="range_apron", init_seconds=0.0)
    span = scheme.intensity_span
    done, t_total, ks = 0, 0.0, []
    for picks, alpha in timed_tfs:
        lut = np.zeros((span, 4))
        lut[:, 3] = alpha
        tf = R.TransferFunction(lut=lut)
        t0 = time.perf_counter()
        sel = R.select_partitions(tf, rscheme)
        R.combine(rset, sel)
        t_total += time.perf_counter() - t0
        done += 1
        ks.append(len(picks))
        if t_total > REF_SAMPLE_S:
            break
    vox = grid.num_blocks * grid.b ** 3
    return {"value": round(vox * done / t_total / 1e9, 4), "unit": "Gvoxel/s", "cores": 1,
            "kind": "reference", "ms_per_step": round(t_total / done * 1e3, 3),
            "sample": f"{done} TF changes (k = {ks[0]}..{ks[-1]}, mean {np.mean(ks):.1f}) of the "
                      f"timed sequence: pdmrender.select_partitions + combine as shipped "
                      f"(baseline/_ref), 1 thread"}


# ---------------------------------------------------------------------------------
# reference arm: the CPU oracle (reference algorithm restated in C) on host cores
# ---------------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle
    from paper_2407_21552_b200 import scheme_uniform
    from paper_2407_21552_b200.synth import synth_boxes

    cfg = CONFIGS[args.config]
    oracle.build()
    threads = oracle.max_threads()
    oracle.set_threads(threads)
    bits, b, n = cfg["bits"], cfg["b"], cfg["n"]
    gdims, (x0, x1), _ = slab_of(cfg, 0, world)
    scheme = scheme_uniform(n, bits)
    bounds = scheme.bounds()
    boxes = synth_boxes(gdims, bits, cfg["seed"], cfg["nbox"])
    t0 = time.perf_counter()
    # the CPU holds the whole job: at weak scaling its per-rank slab (timed
    # once, = the job's throughput), at strong scaling the whole volume
    sdims = (x1 - x0, gdims[1], gdims[2]) if cfg["scaling"] == "weak" else gdims
    if cfg["scaling"] == "weak" and world > 1:
        vox = oracle.synth_volume(bits, gdims, boxes, cfg["seed"], x_range=(x0, x1))
        pdms = oracle.build_pdm_set(vox, b, bounds, cfg["mode"])
        del vox
    else:
        pdms = oracle.build_pdm_set_synth(bits, sdims, boxes, cfg["seed"], b, bounds,
                                          cfg["mode"])
    setup_s = time.perf_counter() - t0
    steps, warm = args.steps, args.warmup
    warm_tfs, timed_tfs = tf_plan(n, bits, steps, warm, cfg["seed"] + 1)
    out = np.empty(pdms.shape[1:], dtype=np.uint8)
    for _, a in warm_tfs:
        oracle.combine(pdms, oracle.select(a, bounds), out=out)
    times = []
    for _, a in timed_tfs:
        t1 = time.perf_counter()
        oracle.combine(pdms, oracle.select(a, bounds), out=out)
        times.append(time.perf_counter() - t1)
    total = sum(times)
    voxels = int(np.prod(sdims))
    val = voxels * steps / total / 1e9
    line = {
        "metric": METRIC,
        "impl": "reference",
        "value": round(val, 3),
        "unit": "Gvoxel/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": round(total / steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (same hash-box volume and TF sequence as the b200 arm)",
        "config": config_keys(cfg, gdims, world),
        "cpu_baseline": {"value": round(val, 3), "unit": "Gvoxel/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{steps} TF changes (select + combine) on the full PDM set "
                                   f"of {sdims}; setup (volume + PDM build) {setup_s:.1f}s "
                                   f"untimed"},
        "e2e": {"value": round(val, 3), "unit": "Gvoxel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_baseline:
        from paper_2407_21552_b200.volume import BlockGrid

        shipped = shipped_reference_sample(pdms, timed_tfs, scheme, BlockGrid.for_dims(sdims, b))
        if shipped is not None:
            line["cpu_baseline"]["shipped_reference"] = shipped
    return line


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c")
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the oracle comparison of the PDMs and every timed D'")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}")
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
