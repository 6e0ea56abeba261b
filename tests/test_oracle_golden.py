"""Pins the CPU oracle (oracle/) against golden vectors produced by running the
reference itself (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import (
    bounds_of,
    chebyshev_oracle,
    golden_case_names,
    load_case,
    load_dt_cases,
    tf_names,
)

CASES = golden_case_names()


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def test_distance_transform_golden():
    for occ, want in load_dt_cases():
        got = oracle.distance_transform(occ)
        assert np.array_equal(got, want), occ.shape


def test_chamfer_empty_is_inf32():
    d = oracle.chamfer_chebyshev(np.zeros((3, 4, 5), dtype=bool))
    assert np.all(d == (1 << 20))


def test_distance_transform_brute_force_small():
    rng = np.random.default_rng(404)
    for _ in range(60):
        dims = tuple(int(rng.integers(1, 9)) for _ in range(3))
        occ = rng.random(dims) < rng.uniform(0.0, 0.6)
        assert np.array_equal(oracle.distance_transform(occ).astype(np.int64),
                              chebyshev_oracle(occ))


@pytest.mark.parametrize("name", CASES)
def test_block_min_max_golden(name):
    c = load_case(name)
    mins, maxs = oracle.block_min_max(c["vox"], int(c["b"]))
    assert np.array_equal(mins, c["mins"]) and np.array_equal(maxs, c["maxs"])


@pytest.mark.parametrize("name", CASES)
def test_partition_occupancy_golden(name):
    c = load_case(name)
    b = int(c["b"])
    bounds = bounds_of(c)
    pres = oracle.partition_presence(c["vox"], b, oracle.pid_lut(bounds), len(bounds))
    assert np.array_equal(pres, c["occ_part_voxel"])
    for p, (lo, hi) in enumerate(bounds):
        assert np.array_equal(oracle.block_any_in_range(c["vox"], b, lo, hi),
                              c["occ_part_voxel"][p])
    ra = oracle.range_apron_presence(c["mins"], c["maxs"], bounds)
    assert np.array_equal(ra, c["occ_part_range_apron"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_build_pdm_set_golden(name, mode):
    c = load_case(name)
    got = oracle.build_pdm_set(c["vox"], int(c["b"]), bounds_of(c), mode)
    assert np.array_equal(got, c[f"pdms_{mode}"])


@pytest.mark.parametrize("name", CASES)
def test_select_combine_tf_golden(name):
    c = load_case(name)
    b = int(c["b"])
    bounds = bounds_of(c)
    for t in tf_names(c):
        alpha = c[f"tf_{t}_alpha"]
        sel = oracle.select(alpha, bounds)
        assert sel == c[f"tf_{t}_sel"].tolist(), t
        for mode in ("voxel", "range_apron"):
            dp = oracle.combine(c[f"pdms_{mode}"], sel)
            assert np.array_equal(dp, c[f"tf_{t}_dprime_{mode}"]), (t, mode)
            lut = np.zeros((alpha.size, 4))
            lut[:, 3] = alpha
            occ = oracle.occupancy_for_tf(c["vox"], b, lut, mode)
            assert np.array_equal(occ, c[f"tf_{t}_occ_{mode}"]), (t, mode)
            std = oracle.standard_distance_map(c["vox"], b, lut, mode)
            assert np.array_equal(std, c[f"tf_{t}_std_{mode}"]), (t, mode)


def test_worked_example_golden():
    from conftest import GOLDEN

    with np.load(GOLDEN / "worked_example.npz") as z:
        bounds = [tuple(map(int, r)) for r in z["bounds"]]
        vox = z["vox"]
        pres = oracle.partition_presence(vox, 1, oracle.pid_lut(bounds), len(bounds))
        pdms = oracle.distance_transform_batch(pres)
        assert np.array_equal(pdms, z["pdms"])
        sel = oracle.select(z["alpha"], bounds)
        assert sel == z["sel"].tolist() == [2, 4]
        assert np.array_equal(oracle.combine(pdms, sel), z["dprime"])


def test_thread_count_does_not_change_results():
    c = load_case("u16_fast_b4_n32")
    oracle.set_threads(1)
    one = oracle.build_pdm_set(c["vox"], int(c["b"]), bounds_of(c), "voxel")
    oracle.set_threads(4)
    four = oracle.build_pdm_set(c["vox"], int(c["b"]), bounds_of(c), "voxel")
    oracle.set_threads(1)
    assert np.array_equal(one, four)


def test_selection_f64_edge_cases():
    bounds = [(0, 63), (64, 127), (128, 191), (192, 255)]
    alpha = np.zeros(256)
    alpha[10] = np.nan  # NaN is transparent
    alpha[70] = 5e-324  # smallest denormal is visible
    alpha[200] = 1e-300
    assert oracle.select(alpha, bounds) == [2, 4]


def test_synth_slab_matches_full():
    from paper_2407_21552_b200.synth import synth_boxes

    dims = (24, 10, 16)
    boxes = synth_boxes(dims, 16, seed=5, nbox=5)
    full = oracle.synth_volume(16, dims, boxes, seed=5)
    part = oracle.synth_volume(16, dims, boxes, seed=5, x_range=(7, 19))
    assert np.array_equal(full[7:19], part)
    assert full.max() > 0 and (full == 0).any()


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
@pytest.mark.parametrize("dims,bits,b,slab", [((37, 9, 11), 16, 4, 8), ((30, 7, 12), 8, 3, 9),
                                               ((16, 5, 6), 8, 2, 2)])
def test_slabwise_synth_build_matches_whole_volume(mode, dims, bits, b, slab):
    """oracle.build_pdm_set_synth (slab-by-slab occupancy, used for the
    2048^3 parity checks) == build_pdm_set on the whole generated volume."""
    from paper_2407_21552_b200.synth import synth_boxes

    boxes = synth_boxes(dims, bits, 5, 6)
    vox = oracle.synth_volume(bits, dims, boxes, 5)
    bounds = [(lo, hi) for lo, hi in _uniform_bounds(5, bits)]
    want = oracle.build_pdm_set(vox, b, bounds, mode)
    got = oracle.build_pdm_set_synth(bits, dims, boxes, 5, b, bounds, mode, slab_voxels=slab)
    assert np.array_equal(got, want)


def _uniform_bounds(n, bits):
    span = 1 << bits
    q, r = divmod(span, n)
    out, lo = [], 0
    for i in range(n):
        w = q + (i < r)
        out.append((lo, lo + w - 1))
        lo += w
    return out
