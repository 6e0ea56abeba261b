"""Generate golden vectors for the distance-map update path by RUNNING THE REFERENCE.

Run here (the container that has /root/reference), never on the GPU box:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``pdmrender`` from /root/reference/pkg/src and its test fixtures from
/root/reference/pkg/tests/conftest.py (random_structured_volume, tf_from_support,
aligned_tf), calls the reference functions on seeded inputs, and writes the
inputs and the reference outputs to tests/golden/cases/*.npz plus a manifest.
The fixtures are committed; tests compare both the CPU oracle (oracle/) and the
CUDA path against them.

Covered (reference file:line in /root/reference/pkg/src/pdmrender):
  distance_transform ............ acceleration.py:177-181 (_kernels.py:17-81)
  block_min_max ................. volume.py:289-300
  occupancy_for_partition ....... acceleration.py:114-142 (both modes)
  occupancy_for_tf .............. acceleration.py:145-174 (both modes)
  standard_distance_map ......... acceleration.py:184-196 (both modes)
  build_pdm_set ................. acceleration.py:199-241 (both modes)
  select_partitions ............. transfer.py:250-259
  combine ....................... acceleration.py:244-276
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import numpy as np  # noqa: E402

import pdmrender as ref  # noqa: E402
from conftest import aligned_tf, random_structured_volume, tf_from_support  # noqa: E402

OUT = Path(__file__).resolve().parent / "cases"


def _tf_set(rng, scheme, bits):
    """A mix of TFs: random support, aligned, archetypes, empty, NaN/denormal edge cases."""
    length = 1 << bits
    tfs = {}
    if bits == 8:
        for p in (0.02, 0.1, 0.5):
            tfs[f"rand{p}"] = tf_from_support(rng.random(length) < p, rng)
    else:
        # 16-bit: random bands (per-intensity random support selects every partition)
        for t in range(3):
            support = np.zeros(length, dtype=bool)
            for _ in range(int(rng.integers(1, 4))):
                lo = int(rng.integers(0, length))
                hi = min(length, lo + int(rng.integers(1, length // 8)))
                support[lo:hi] = True
            tfs[f"band{t}"] = tf_from_support(support, rng)
    k = int(rng.integers(1, scheme.n + 1))
    picks = set(int(i) for i in rng.choice(np.arange(1, scheme.n + 1), size=k, replace=False))
    tfs["aligned"] = aligned_tf(scheme, picks, rng)
    for name in ("tf1", "tf3", "tf4"):
        tfs[name] = ref.tf_archetype(name, bits)
    tfs["empty"] = ref.TransferFunction(lut=np.zeros((length, 4)))
    lut = np.zeros((length, 4))
    lut[int(rng.integers(0, length)), 3] = np.nan  # NaN passes validation, is transparent
    lut[int(rng.integers(0, length)), 3] = 5e-324  # denormal is visible
    tfs["nan_denormal"] = ref.TransferFunction(lut=lut)
    return tfs


def volume_case(name, rng, dims, bits, b, n, scheme_kind="uniform"):
    vol = random_structured_volume(rng, dims, bits)
    grid = ref.BlockGrid.for_dims(vol.dims, b)
    if scheme_kind == "uniform":
        scheme = ref.scheme_uniform(n, bits)
    else:
        rho = int(np.bincount(vol.voxels.ravel().astype(np.int64)).argmax())
        rho = min(rho, (1 << bits) - n)
        scheme = ref.scheme_with_min_special(n, bits, rho)
    rec = {
        "vox": vol.voxels,
        "b": np.int64(b),
        "bounds": np.array(scheme.bounds(), dtype=np.int64),
    }
    mins, maxs = ref.block_min_max(vol, grid)
    rec["mins"], rec["maxs"] = mins, maxs
    for mode in ("voxel", "range_apron"):
        occ = np.stack([ref.occupancy_for_partition(vol, grid, p, mode).occupied
                        for p in scheme.partitions])
        rec[f"occ_part_{mode}"] = occ
        pset = ref.build_pdm_set(vol, grid, scheme, mode)
        rec[f"pdms_{mode}"] = np.stack([d.dist for d in pset.pdms])
    tfs = _tf_set(rng, scheme, bits)
    rec["tf_names"] = np.array(list(tfs.keys()))
    pset_v = ref.build_pdm_set(vol, grid, scheme, "voxel")
    pset_r = ref.build_pdm_set(vol, grid, scheme, "range_apron")
    for tname, tf in tfs.items():
        rec[f"tf_{tname}_alpha"] = tf.lut[:, 3].copy()
        sel = ref.select_partitions(tf, scheme)
        rec[f"tf_{tname}_sel"] = np.array(sel.sorted, dtype=np.int64)
        rec[f"tf_{tname}_dprime_voxel"] = ref.combine(pset_v, sel).dist
        rec[f"tf_{tname}_dprime_range_apron"] = ref.combine(pset_r, sel).dist
        for mode in ("voxel", "range_apron"):
            rec[f"tf_{tname}_occ_{mode}"] = ref.occupancy_for_tf(vol, grid, tf, mode).occupied
            rec[f"tf_{tname}_std_{mode}"] = ref.standard_distance_map(vol, grid, tf, mode).dist
    np.savez_compressed(OUT / f"vol_{name}.npz", **rec)
    return {"name": name, "dims": list(dims), "bits": bits, "b": b, "n": n,
            "scheme": scheme_kind, "tfs": list(tfs.keys())}


def dt_cases(rng):
    occs, dists = [], []
    shapes = [tuple(int(rng.integers(1, 11)) for _ in range(3)) for _ in range(120)]
    for i, sh in enumerate(shapes):
        dens = (0.0, 1.0, 0.002, 0.05, 0.3)[i % 5]
        occ = rng.random(sh) < dens
        occs.append(occ)
    for sh, pts in (((300, 1, 1), [(0, 0, 0)]), ((1, 300, 2), [(0, 299, 1)]),
                    ((2, 3, 600), [(1, 2, 0), (0, 0, 590)]), ((270, 5, 4), [(3, 4, 3)]),
                    ((9, 9, 9), [(4, 4, 4)]), ((40, 33, 70), [(0, 0, 0), (39, 32, 69)])):
        occ = np.zeros(sh, dtype=bool)
        for p in pts:
            occ[p] = True
        occs.append(occ)
    occs.append(rng.random((64, 48, 80)) < 0.0005)
    occs.append(rng.random((33, 65, 17)) < 0.01)
    for occ in occs:
        dm = ref.distance_transform(ref.OccupancyMap(b=1, bdims=occ.shape, occupied=occ))
        dists.append(dm.dist)
    rec = {}
    for i, (o, d) in enumerate(zip(occs, dists)):
        rec[f"occ_{i}"] = o
        rec[f"dist_{i}"] = d
    rec["count"] = np.int64(len(occs))
    np.savez_compressed(OUT / "dt.npz", **rec)
    return len(occs)


def worked_example():
    """test_acceptance.py:92-156 Fig. 1 chain at b=1, 3-bit intensities."""
    vox = np.zeros((6, 6, 1), dtype=np.uint8)
    vox[1, 1, 0] = 3
    vox[2, 1, 0] = 6
    vox[1, 2, 0] = 6
    vox[2, 2, 0] = 7
    vox[5, 5, 0] = 2
    vol = ref.Volume.from_array(vox)
    grid = ref.BlockGrid.for_dims((6, 6, 1), 1)
    scheme = ref.scheme_uniform(4, bits=3)
    pdms = tuple(ref.distance_transform(ref.occupancy_for_partition(vol, grid, p, "voxel"))
                 for p in scheme.partitions)
    sup = np.zeros(8, dtype=bool)
    sup[[2, 3, 6, 7]] = True
    tf = tf_from_support(sup)
    sel = ref.select_partitions(tf, scheme)
    pset = ref.PdmSet(grid=grid, scheme=scheme, pdms=pdms, occupancy_mode="voxel",
                      init_seconds=0.0)
    np.savez_compressed(OUT / "worked_example.npz", vox=vox, bounds=np.array(scheme.bounds()),
                        pdms=np.stack([d.dist for d in pdms]), alpha=tf.lut[:, 3].copy(),
                        sel=np.array(sel.sorted), dprime=ref.combine(pset, sel).dist)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(2407_21552)
    manifest = {"reference": "pdmrender " + ref.__version__, "numpy": np.__version__,
                "cases": []}
    manifest["dt_grids"] = dt_cases(rng)
    worked_example()
    specs = [
        # name, dims, bits, b, n, scheme
        ("u8_partial_b4", (13, 9, 11), 8, 4, 8, "uniform"),
        ("u8_partial_b3", (12, 5, 9), 8, 3, 4, "uniform"),
        ("u8_odd_b2", (9, 13, 6), 8, 2, 16, "uniform"),
        ("u8_b1", (7, 6, 5), 8, 1, 8, "uniform"),
        ("u8_b7", (17, 3, 20), 8, 7, 5, "uniform"),
        ("u8_n1", (12, 12, 12), 8, 4, 1, "uniform"),
        ("u8_n100_minspecial", (20, 18, 22), 8, 2, 100, "min_special"),
        ("u8_n64_b4", (24, 20, 32), 8, 4, 64, "uniform"),
        ("u8_fast_b4", (40, 36, 64), 8, 4, 32, "uniform"),
        ("u8_fast_b8", (48, 40, 64), 8, 8, 16, "min_special"),
        ("u8_fast_b16", (33, 32, 48), 8, 16, 8, "uniform"),
        ("u8_n256_b2", (10, 12, 16), 8, 2, 256, "uniform"),
        ("u16_partial_b4", (13, 11, 12), 16, 4, 8, "uniform"),
        ("u16_b8_n16", (24, 17, 30), 16, 8, 16, "uniform"),
        ("u16_n32_b4", (22, 20, 24), 16, 4, 32, "min_special"),
        ("u16_fast_b4_n32", (40, 44, 64), 16, 4, 32, "uniform"),
        ("u16_fast_b8_n16", (48, 40, 64), 16, 8, 16, "uniform"),
        ("u16_fast_b2_n64", (20, 18, 32), 16, 2, 64, "uniform"),
        ("u16_n33", (16, 16, 24), 16, 4, 33, "uniform"),
        ("u16_b1_n4", (6, 7, 16), 16, 1, 4, "uniform"),
    ]
    for name, dims, bits, b, n, kind in specs:
        manifest["cases"].append(volume_case(name, rng, dims, bits, b, n, kind))
        print("wrote", name, flush=True)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main()
