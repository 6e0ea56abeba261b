"""Property and edge-case tests of the CUDA path (needs a B200).

* hypothesis: DT vs the all-pairs oracle on random small grids; POM/PDM build
  and select+merge vs the C oracle on random volumes / schemes / TFs;
* large-n paths: n in {100, 300, 1000} at 8 and 16 bits (multi-word masks,
  global-atomic POM, >240-map merges in passes, device flags up to 4096);
* degenerate shapes: single voxel, single block, 1-long axes, b > dims;
* full-size properties at BASELINE config c (1024^3): PDM zero set == POM,
  1-Lipschitz along every axis, merge == min of the selected planes, and
  combine(S1 u S2) == min(combine(S1), combine(S2)).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_2407_21552_b200 as pdm
from conftest import chebyshev_oracle, lut_from_support, random_structured_volume

pytestmark = pytest.mark.gpu
SETTINGS = settings(max_examples=40, deadline=None,
                    suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])


@SETTINGS
@given(dims=st.tuples(*(st.integers(1, 9) for _ in range(3))), seed=st.integers(0, 10**6),
       density=st.floats(0.0, 1.0))
def test_dt_property(dims, seed, density):
    occ = np.random.default_rng(seed).random(dims) < density
    dm = pdm.distance_transform(pdm.OccupancyMap(b=1, bdims=dims, occupied=occ))
    assert np.array_equal(dm.dist.astype(np.int64), chebyshev_oracle(occ))


@SETTINGS
@given(data=st.data())
def test_build_select_merge_property(data):
    bits = data.draw(st.sampled_from([8, 16]))
    dims = tuple(data.draw(st.integers(1, 26)) for _ in range(3))
    b = data.draw(st.sampled_from([1, 2, 3, 4, 8]))
    n = data.draw(st.integers(1, 70))
    mode = data.draw(st.sampled_from(["voxel", "range_apron"]))
    seed = data.draw(st.integers(0, 10**6))
    rng = np.random.default_rng(seed)
    vox = random_structured_volume(rng, dims, bits)
    scheme = pdm.scheme_uniform(n, bits)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, b), scheme,
                             mode)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
    assert np.array_equal(np.stack([d.dist for d in pset.pdms]), want)
    span = 1 << bits
    lut = lut_from_support(rng.random(span) < data.draw(st.floats(0.0, 0.01 if bits == 16 else 0.5)),
                           rng)
    sel = pdm.select_partitions(pdm.TransferFunction(lut=lut), scheme)
    assert sel.sorted == oracle.select(lut[:, 3], scheme.bounds())
    assert np.array_equal(pdm.combine(pset, sel).dist, oracle.combine(want, sel.sorted))


@pytest.mark.parametrize("bits,n,dims,b", [
    (8, 100, (20, 18, 32), 2), (8, 256, (16, 16, 32), 4), (16, 300, (24, 20, 32), 4),
    (16, 1000, (16, 12, 24), 2), (16, 5000, (12, 8, 16), 2),
])
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_large_partition_counts(bits, n, dims, b, mode):
    rng = np.random.default_rng(n + bits)
    vox = random_structured_volume(rng, dims, bits)
    scheme = pdm.scheme_uniform(n, bits)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, b), scheme,
                             mode)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
    assert np.array_equal(np.stack([d.dist for d in pset.pdms]), want)
    for p in (0.001, 0.05, 1.0):
        lut = lut_from_support(rng.random(1 << bits) < p, rng)
        tf = pdm.TransferFunction(lut=lut)
        sel = pdm.select_partitions(tf, scheme)
        ref = oracle.select(lut[:, 3], scheme.bounds())
        assert sel.sorted == ref
        assert np.array_equal(pdm.combine(pset, sel).dist, oracle.combine(want, ref))
        if n <= 4096:
            assert np.array_equal(pdm.update_from_tf(pset, tf).dist, oracle.combine(want, ref))


@pytest.mark.parametrize("dims,b", [((1, 1, 1), 1), ((1, 1, 1), 4), ((3, 1, 1), 8), ((1, 5, 1), 2),
                                    ((1, 1, 37), 4), ((2, 3, 4), 16), ((7, 1, 300), 1)])
@pytest.mark.parametrize("bits", [8, 16])
def test_degenerate_shapes(dims, b, bits):
    rng = np.random.default_rng(sum(dims) * b + bits)
    vox = rng.integers(0, 1 << bits, size=dims).astype(np.uint8 if bits == 8 else np.uint16)
    vox[rng.random(dims) < 0.7] = 0
    scheme = pdm.scheme_uniform(4, bits)
    vol = pdm.Volume.from_array(vox)
    grid = pdm.BlockGrid.for_dims(dims, b)
    for mode in ("voxel", "range_apron"):
        pset = pdm.build_pdm_set(vol, grid, scheme, mode)
        want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
        assert np.array_equal(np.stack([d.dist for d in pset.pdms]), want), mode
    mins, maxs = pdm.block_min_max(vol, grid)
    omin, omax = oracle.block_min_max(vox, b)
    assert np.array_equal(mins, omin) and np.array_equal(maxs, omax)


@pytest.fixture(scope="module")
def config_c():
    from paper_2407_21552_b200 import synth

    vol = synth.synth_volume_device((1024, 1024, 1024), 16, seed=2407, nbox=12)
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    scheme = pdm.scheme_uniform(32, 16)
    pset = pdm.build_pdm_set(vol, grid, scheme, "range_apron")
    mask = pdm.partition_mask(vol, grid, scheme, "range_apron")
    return vol, grid, scheme, pset, mask


def test_full_size_pdm_properties(config_c):
    vol, grid, scheme, pset, mask = config_c
    nb = grid.num_blocks
    st_ = pset.storage[:, :nb]
    bits = mask[:, 0].view(torch.int32)
    for p in range(scheme.n):
        plane = st_[p].view(grid.bdims).to(torch.int16)
        occ = ((bits >> p) & 1).bool().view(grid.bdims)
        assert torch.equal(plane == 0, occ), p  # zero set == POM
        for ax in range(3):  # 1-Lipschitz
            assert int(plane.diff(dim=ax).abs().max()) <= 1, (p, ax)


def test_full_size_merge_properties(config_c):
    vol, grid, scheme, pset, _ = config_c
    nb = grid.num_blocks
    planes = pset.storage[:, :nb]
    rng = np.random.default_rng(1)
    s1 = set(int(i) for i in rng.choice(np.arange(1, 33), 7, replace=False))
    s2 = set(int(i) for i in rng.choice(np.arange(1, 33), 11, replace=False))
    sel = lambda s: pdm.PartitionSelection(selected=frozenset(s), n=32)  # noqa: E731
    d1 = pdm.combine(pset, sel(s1)).device().view(-1)
    d2 = pdm.combine(pset, sel(s2)).device().view(-1)
    d12 = pdm.combine(pset, sel(s1 | s2)).device().view(-1)
    assert torch.equal(d12, torch.minimum(d1, d2))
    want = planes[[i - 1 for i in sorted(s1)]].min(dim=0).values
    assert torch.equal(d1, want)
    assert torch.equal(pdm.combine(pset, sel(set())).device(),
                       torch.full(grid.bdims, 255, dtype=torch.uint8, device="cuda"))


def test_full_size_dt_spot_check(config_c):
    """Exact distance for sampled near cells by brute force in a window."""
    vol, grid, scheme, pset, mask = config_c
    nb = grid.num_blocks
    bits = mask[:, 0].view(torch.int32)
    rng = np.random.default_rng(3)
    for p in (0, 5, 17, 31):
        plane = pset.storage[p, :nb].view(grid.bdims)
        occ = ((bits >> p) & 1).bool().view(grid.bdims)
        near = torch.nonzero((plane > 0) & (plane <= 6))
        if near.shape[0] == 0:
            continue
        for idx in near[torch.from_numpy(rng.choice(near.shape[0], min(64, near.shape[0]),
                                                    replace=False))].tolist():
            d = int(plane[tuple(idx)])
            lo = [max(0, c - d) for c in idx]
            hi = [min(s, c + d + 1) for c, s in zip(idx, grid.bdims)]
            win = occ[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
            assert bool(win.any()), (p, idx, d)  # something at distance <= d
            lo1 = [max(0, c - d + 1) for c in idx]
            hi1 = [min(s, c + d) for c, s in zip(idx, grid.bdims)]
            assert not bool(occ[lo1[0]:hi1[0], lo1[1]:hi1[1], lo1[2]:hi1[2]].any()), (p, idx, d)
