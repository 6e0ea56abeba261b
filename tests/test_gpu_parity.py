"""GPU parity: the CUDA path (through the drop-in API, hence the C ABI) against
the reference's golden vectors and the CPU oracle, bit-exact.  Needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2407_21552_b200 as pdm
from conftest import (
    GOLDEN,
    bounds_of,
    chebyshev_oracle,
    golden_case_names,
    load_case,
    load_dt_cases,
    lut_from_support,
    random_structured_volume,
    tf_names,
)

pytestmark = pytest.mark.gpu
CASES = golden_case_names()


def _scheme(bounds):
    return pdm.PartitionScheme(tuple(pdm.Partition(lo, hi) for lo, hi in bounds))


def _tf(alpha):
    lut = np.zeros((alpha.size, 4))
    lut[:, 3] = alpha
    return pdm.TransferFunction(lut=lut)


def _stack(pset):
    return np.stack([d.dist for d in pset.pdms])


# --- distance transform --------------------------------------------------------------

def test_distance_transform_golden():
    for occ, want in load_dt_cases():
        dm = pdm.distance_transform(pdm.OccupancyMap(b=1, bdims=occ.shape, occupied=occ))
        assert np.array_equal(dm.dist, want), occ.shape


def test_distance_transform_brute_force():
    rng = np.random.default_rng(404)
    for case in range(200):
        dims = tuple(int(rng.integers(1, 11)) for _ in range(3))
        occ = (np.zeros(dims, bool) if case == 0 else np.ones(dims, bool) if case == 1
               else rng.random(dims) < rng.uniform(0.0, 0.6))
        dm = pdm.distance_transform(pdm.OccupancyMap(b=1, bdims=dims, occupied=occ))
        assert np.array_equal(dm.dist.astype(np.int64), chebyshev_oracle(occ)), dims


def test_distance_transform_clamp_far_field():
    occ = np.zeros((300, 1, 1), bool)
    occ[0] = True
    d = pdm.distance_transform(pdm.OccupancyMap(b=4, bdims=occ.shape, occupied=occ)).dist
    assert d[254, 0, 0] == 254 and d[255, 0, 0] == 255 and d[299, 0, 0] == 255
    for shape, pt in (((2, 700, 3), (1, 3, 2)), ((3, 2, 1100), (0, 1, 1099)),
                      ((5, 1300, 1), (4, 0, 0))):
        occ = np.zeros(shape, bool)
        occ[pt] = True
        got = pdm.distance_transform(pdm.OccupancyMap(b=1, bdims=shape, occupied=occ)).dist
        assert np.array_equal(got, oracle.distance_transform(occ)), shape


def test_distance_transform_random_vs_oracle_medium():
    rng = np.random.default_rng(9)
    for dims, dens in (((64, 48, 80), 0.0005), ((33, 65, 17), 0.01), ((70, 70, 70), 0.00002),
                       ((16, 300, 40), 0.001), ((128, 96, 260), 0.000005)):
        occ = rng.random(dims) < dens
        got = pdm.distance_transform(pdm.OccupancyMap(b=1, bdims=dims, occupied=occ)).dist
        assert np.array_equal(got, oracle.distance_transform(occ)), dims


@pytest.mark.parametrize("dims", [
    (12, 128, 256),  # y strided with 16-byte tile copies, z swizzled 16-byte rows
    (9, 256, 128),   # swizzled rows of 128
    (7, 100, 48),    # 16-byte strided copies, padded rows (48 % 128 != 0)
    (6, 61, 20),     # 4-byte copies, odd line length
    (5, 30, 13),     # scalar tile copies, partial warp tiles
    (300, 3, 256),   # x lines > 256 blocks (dist1d) with swizzled z rows
    (4, 300, 384),   # 257..512-long lines: 16-bit sweep tables, strided y, swizzled z rows
    (3, 257, 301),   # odd 16-bit-table lengths: padded rows, scalar steps
    (2, 512, 512),   # longest sweep lines
    (3, 256, 256),   # TMEM sweeps: y and z lines of 256 in full tiles
    (2, 256, 96),    # TMEM y sweep (bz = 96), padded-row z tiles
    (5, 64, 256),    # TMEM z sweep with fused packing rows, strided y of 64
    (2, 512, 96),    # TMEM y sweep of 512-long lines
])
def test_distance_transform_tile_layouts(dims):
    """Every shared-memory tile layout of the sweep envelope kernel against
    the oracle, with far fields (values reaching the 255 clamp) and clusters."""
    rng = np.random.default_rng(sum(dims))
    for dens in (0.0, 0.00003, 0.002, 0.05):
        occ = rng.random(dims) < dens
        if dens == 0.0:
            occ[tuple(int(rng.integers(0, d)) for d in dims)] = True
        got = pdm.distance_transform(pdm.OccupancyMap(b=1, bdims=dims, occupied=occ)).dist
        assert np.array_equal(got, oracle.distance_transform(occ)), (dims, dens)


# --- golden volume cases ---------------------------------------------------------------

@pytest.fixture(scope="module", params=CASES)
def case(request):
    c = load_case(request.param)
    vol = pdm.Volume.from_array(c["vox"])
    grid = pdm.BlockGrid.for_dims(vol.dims, int(c["b"]))
    return c, vol, grid, _scheme(bounds_of(c))


def test_block_min_max(case):
    c, vol, grid, _ = case
    mins, maxs = pdm.block_min_max(vol, grid)
    assert mins.dtype == c["mins"].dtype
    assert np.array_equal(mins, c["mins"]) and np.array_equal(maxs, c["maxs"])


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_occupancy_for_partition(case, mode):
    c, vol, grid, scheme = case
    mm = pdm.block_min_max_device(vol, grid) if mode == "range_apron" else None
    for p, part in enumerate(scheme.partitions):
        occ = pdm.occupancy_for_partition(vol, grid, part, mode, minmax=mm)
        assert np.array_equal(occ.occupied, c[f"occ_part_{mode}"][p]), p


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_build_pdm_set(case, mode):
    c, vol, grid, scheme = case
    pset = pdm.build_pdm_set(vol, grid, scheme, mode)
    assert pset.n == scheme.n and pset.occupancy_mode == mode and pset.init_seconds > 0
    assert np.array_equal(_stack(pset), c[f"pdms_{mode}"])


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_select_combine_and_recompute(case, mode):
    c, vol, grid, scheme = case
    pset = pdm.build_pdm_set(vol, grid, scheme, mode)
    for t in tf_names(c):
        tf = _tf(c[f"tf_{t}_alpha"])
        sel = pdm.select_partitions(tf, scheme)
        assert sel.sorted == c[f"tf_{t}_sel"].tolist(), t
        dp = pdm.combine(pset, sel)
        assert np.array_equal(dp.dist, c[f"tf_{t}_dprime_{mode}"]), (t, mode)
        fused = pdm.update_from_tf(pset, tf)
        assert np.array_equal(fused.dist, c[f"tf_{t}_dprime_{mode}"]), (t, mode)
        occ = pdm.occupancy_for_tf(vol, grid, tf, mode)
        assert np.array_equal(occ.occupied, c[f"tf_{t}_occ_{mode}"]), (t, mode)
        std = pdm.standard_distance_map(vol, grid, tf, mode)
        assert np.array_equal(std.dist, c[f"tf_{t}_std_{mode}"]), (t, mode)


def test_fused_recompute_matches_composition(case):
    """standard_distance_map runs fused (occupancy written as the DT seed);
    it must equal distance_transform(occupancy_for_tf(...)) and the golden,
    with minmax omitted, given on the device, or given as host arrays."""
    c, vol, grid, _ = case
    mm_dev = pdm.block_min_max_device(vol, grid)
    mm_host = pdm.block_min_max(vol, grid)
    for t in tf_names(c):
        tf = _tf(c[f"tf_{t}_alpha"])
        for mode in ("voxel", "range_apron"):
            want = c[f"tf_{t}_std_{mode}"]
            comp = pdm.distance_transform(pdm.occupancy_for_tf(vol, grid, tf, mode))
            assert np.array_equal(comp.dist, want), (t, mode)
            for mm in (None, mm_dev, mm_host):
                got = pdm.standard_distance_map(vol, grid, tf, mode, minmax=mm)
                assert np.array_equal(got.dist, want), (t, mode, type(mm))


def test_recompute_minmax_shape_mismatch():
    vol = pdm.Volume.from_array(np.zeros((8, 8, 8), np.uint8))
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    bad = (np.zeros((2, 2, 1), np.uint8), np.zeros((2, 2, 1), np.uint8))
    tf = pdm.tf_archetype("tf1", 8)
    with pytest.raises(ValueError):
        pdm.standard_distance_map(vol, grid, tf, "range_apron", minmax=bad)
    with pytest.raises(ValueError):
        pdm.occupancy_for_tf(vol, grid, tf, "range_apron", minmax=bad)


@pytest.mark.parametrize("span", [1, 7, 1024, 1025, 8191, 8192, 8193, 40000, 65536])
def test_alpha_support_kernel(span):
    """pdm_alpha_support against numpy: nz = alpha > 0 (NaN transparent,
    denormals visible) and prefix = [0] + cumsum(nz) (acceleration.py:166,171),
    for spans that end inside a tile, on a tile and on a batch boundary, and
    for a strided alpha (the LUT's column 3)."""
    import torch

    from paper_2407_21552_b200 import _lib

    rng = np.random.default_rng(span)
    lut = np.zeros((span, 4))
    a = np.where(rng.random(span) < 0.3, rng.random(span), 0.0)
    a[rng.random(span) < 0.01] = np.nan
    a[rng.random(span) < 0.01] = 5e-324
    lut[:, 3] = a
    L = _lib.lib()
    dev = torch.from_numpy(lut).cuda()
    alpha = dev[:, 3]
    nz = torch.empty(span, dtype=torch.uint8, device="cuda")
    prefix = torch.full((span + 1,), -1, dtype=torch.int32, device="cuda")
    _lib.check(L.pdm_alpha_support(_lib.ptr(alpha), span, alpha.stride(0), _lib.ptr(nz),
                                   _lib.ptr(prefix), _lib.stream_handle()), "alpha_support")
    want = (a > 0.0).astype(np.uint8)
    assert np.array_equal(nz.cpu().numpy(), want)
    assert np.array_equal(prefix.cpu().numpy(), np.concatenate(([0], np.cumsum(want))))
    nz2 = torch.empty(span, dtype=torch.uint8, device="cuda")
    _lib.check(L.pdm_alpha_support(_lib.ptr(alpha), span, alpha.stride(0), _lib.ptr(nz2), None,
                                   _lib.stream_handle()), "alpha_support")
    assert np.array_equal(nz2.cpu().numpy(), want)


def test_worked_example():
    with np.load(GOLDEN / "worked_example.npz") as z:
        scheme = _scheme([tuple(map(int, r)) for r in z["bounds"]])
        vol = pdm.Volume.from_array(z["vox"])
        grid = pdm.BlockGrid.for_dims(vol.dims, 1)
        # 3-bit scheme over a uint8 volume: built per partition as in
        # test_acceptance.py:121-128 (build_pdm_set would reject the span)
        pdms = tuple(pdm.distance_transform(pdm.occupancy_for_partition(vol, grid, p, "voxel"))
                     for p in scheme.partitions)
        pset = pdm.PdmSet(grid=grid, scheme=scheme, pdms=pdms, occupancy_mode="voxel")
        assert np.array_equal(_stack(pset), z["pdms"])
        sel = pdm.select_partitions(_tf(z["alpha"]), scheme)
        assert sel.sorted == [2, 4]
        assert np.array_equal(pdm.combine(pset, sel).dist, z["dprime"])


# --- combine semantics (acceleration.py:244-276) ----------------------------------------

@pytest.fixture(scope="module")
def built16():
    rng = np.random.default_rng(6)
    vol = pdm.Volume.from_array(random_structured_volume(rng, (16, 16, 16)))
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    scheme = pdm.scheme_uniform(16, 8)
    return scheme, pdm.build_pdm_set(vol, grid, scheme, "voxel")


def test_combine_empty_singleton_full(built16):
    scheme, pset = built16
    sel = lambda s: pdm.PartitionSelection(selected=frozenset(s), n=scheme.n)  # noqa: E731
    assert np.all(pdm.combine(pset, sel(())).dist == 255)
    single = pdm.combine(pset, sel({3}))
    assert np.array_equal(single.dist, pset.pdms[2].dist)
    assert single.device().data_ptr() != pset.pdms[2].device().data_ptr()
    full = pdm.combine(pset, sel(range(1, 17)))
    assert np.array_equal(full.dist, np.minimum.reduce([p.dist for p in pset.pdms]))
    for chunk in (1, 2, 3, 100):
        s = sel({1, 4, 7, 9, 15})
        assert np.array_equal(pdm.combine(pset, s).dist,
                              pdm.combine(pset, s, max_maps_per_pass=chunk).dist)
    with pytest.raises(ValueError):
        pdm.combine(pset, sel({1}), max_maps_per_pass=0)
    small = pdm.combine(pset, sel({2, 5})).dist
    large = pdm.combine(pset, sel({2, 5, 9, 12})).dist
    assert np.all(large <= small)


def test_combine_is_eager_and_host_view_lazy(built16):
    """combine() returns a finished map (the reference's contract,
    acceleration.py:244-276): its merge has run into a fresh HBM buffer and
    the stream is idle when it returns; .dist then makes the host view.  Every
    selection kind (device flags, host indices, empty), both access orders."""
    import torch

    scheme, pset = built16
    want = np.minimum.reduce([pset.pdms[i - 1].dist for i in (2, 7, 11)])
    lut = np.zeros((256, 4))
    for i in (2, 7, 11):
        lo, hi = scheme.partitions[i - 1].rho_lo, scheme.partitions[i - 1].rho_hi
        lut[lo: hi + 1, 3] = 0.5
    tf = pdm.TransferFunction(lut=lut)
    sel = pdm.select_partitions(tf, scheme)
    assert torch.cuda.current_stream().query()  # selection complete on return
    a = pdm.combine(pset, sel)  # host selection (select_partitions)
    assert a._dev is not None and a._host is None
    assert torch.cuda.current_stream().query()  # merge complete on return
    assert np.array_equal(a.dist, want) and np.array_equal(a.device().cpu().numpy(), want)
    b = pdm.combine(pset, pdm.select_partitions(tf, scheme))  # device view first
    assert np.array_equal(b.device().cpu().numpy(), want) and np.array_equal(b.dist, want)
    flags = pdm.select_partitions_device(pdm.transfer.alpha_to_device(tf), scheme)
    f = pdm.combine(pset, pdm.PartitionSelection(n=16, flags_dev=flags))  # device flags
    assert torch.cuda.current_stream().query()
    assert np.array_equal(f.dist, want) and f.dist.ctypes.data != b.dist.ctypes.data
    c = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset({2, 7, 11}), n=16))
    assert torch.cuda.current_stream().query()
    assert np.array_equal(c.dist, want)
    e = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset(), n=16))
    assert np.all(e.dist == 255) and int(e.device().min()) == 255
    assert a.dist.ctypes.data != b.dist.ctypes.data
    for p in pset.pdms:  # never aliases a PDM
        assert a.device().data_ptr() != p.device().data_ptr()


def test_select_rereads_a_mutated_lut(built16):
    """select_partitions stages tf.lut on every call (the reference re-reads
    it): an in-place edit of the LUT changes the next selection."""
    scheme, _ = built16
    lut = np.zeros((256, 4))
    lut[3, 3] = 0.5
    tf = pdm.TransferFunction(lut=lut)
    assert pdm.select_partitions(tf, scheme).sorted == [1]
    tf.lut[3, 3] = 0.0
    tf.lut[255, 3] = 0.25
    assert pdm.select_partitions(tf, scheme).sorted == [16]


@pytest.mark.parametrize("fmt", [1, 2, 3])
def test_dprime_to_host_formats_and_pieces(fmt):
    """pdm_dprime_to_host through the C ABI: a finished D' in HBM re-encoded
    in the nibble, delta and sparse delta forms, 1-7 pieces, 1-Lipschitz maps
    with zero plateaus, flat runs and slopes, sizes with a partial last item;
    bytes past map_bytes are never written."""
    import torch

    from paper_2407_21552_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(10 + fmt)
    st = _lib.stream_handle()
    for map_bytes in (70000, 4096 * 3 + 5, 31, 1):
        steps = rng.choice([-1, 0, 0, 0, 1], size=map_bytes)
        d = np.clip(int(rng.integers(0, 40)) + np.cumsum(steps), 0, 255)
        d[: map_bytes // 5] = 0
        d[map_bytes // 5:] = np.minimum(d[map_bytes // 5:],
                                         np.arange(1, map_bytes - map_bytes // 5 + 1))
        d = d.astype(np.uint8)
        assert map_bytes < 2 or np.abs(np.diff(d.astype(np.int16))).max() <= 1
        dev = torch.from_numpy(d).cuda()
        chunks = int(L.pdm_packed_chunks(map_bytes))
        stage = torch.empty(max(chunks * 8, -(-chunks // 64) * 336), dtype=torch.uint8,
                            pin_memory=True)
        stage_b = torch.empty(chunks, dtype=torch.uint8, pin_memory=True)
        for pieces in (1, 3, 7):
            out = np.full(map_bytes + 32, 0xCD, np.uint8)
            _lib.check(L.pdm_dprime_to_host(_lib.ptr(dev), map_bytes, stage.data_ptr(),
                                            stage_b.data_ptr(), out.ctypes.data, pieces, fmt,
                                            st), "dprime_to_host")
            assert np.array_equal(out[:map_bytes], d), (map_bytes, pieces)
            assert (out[map_bytes:] == 0xCD).all()
    out = np.empty(64, np.uint8)
    with pytest.raises(ValueError):
        _lib.check(L.pdm_dprime_to_host(_lib.ptr(dev), 1, stage.data_ptr(), stage_b.data_ptr(),
                                        out.ctypes.data, 1, 4, st), "bad format")


def test_combine_more_than_one_param_batch():
    rng = np.random.default_rng(3)
    vox = random_structured_volume(rng, (12, 10, 16), bits=8)
    vol = pdm.Volume.from_array(vox)
    grid = pdm.BlockGrid.for_dims(vol.dims, 2)
    scheme = pdm.scheme_uniform(256, 8)
    pset = pdm.build_pdm_set(vol, grid, scheme, "voxel")
    want = oracle.build_pdm_set(vox, 2, scheme.bounds(), "voxel")
    assert np.array_equal(_stack(pset), want)
    for k in (239, 240, 241, 256):
        s = sorted(rng.choice(np.arange(1, 257), size=k, replace=False).tolist())
        got = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset(s), n=256)).dist
        assert np.array_equal(got, oracle.combine(want, s)), k


def test_combine_rebuilt_from_host_maps(built16):
    scheme, pset = built16
    host = pdm.PdmSet(grid=pset.grid, scheme=scheme,
                      pdms=tuple(pdm.DistanceMap(4, pset.grid.bdims, d.dist.copy())
                                 for d in pset.pdms), occupancy_mode="voxel")
    s = pdm.PartitionSelection(selected=frozenset({2, 9, 16}), n=16)
    assert np.array_equal(pdm.combine(host, s).dist, pdm.combine(pset, s).dist)


def test_pdm_set_round_trip(tmp_path, built16):
    scheme, pset = built16
    pdm.save_pdm_set(pset, tmp_path / "set.bin")
    back = pdm.load_pdm_set(tmp_path / "set.bin")
    assert back.n == pset.n and back.grid == pset.grid and back.scheme.bounds() == scheme.bounds()
    assert np.array_equal(_stack(back), _stack(pset))


# --- random fast-path shapes vs the oracle -----------------------------------------------

@pytest.mark.parametrize("dims,bits,b,n", [
    ((64, 64, 128), 16, 4, 32), ((48, 40, 64), 16, 8, 16), ((40, 36, 96), 8, 4, 64),
    ((37, 29, 64), 16, 2, 33), ((31, 17, 48), 8, 16, 8), ((20, 20, 24), 16, 1, 4),
    ((65, 33, 40), 16, 4, 64),
    # TMA apron planes (16-bit, b = 4): three strips with a partial last one
    # (nz = 520) and a partial last block row; ny = 5 < 6 keeps the cp.async ring
    ((13, 23, 520), 16, 4, 16), ((11, 5, 264), 16, 4, 8),
    # pass x from the mask with x lines of 257..512 blocks (one CTA per SM)
    ((1200, 8, 128), 16, 4, 16), ((2040, 4, 128), 16, 4, 32),
])
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_random_volumes_vs_oracle(dims, bits, b, n, mode):
    rng = np.random.default_rng(sum(dims) + bits + b + n)
    vox = random_structured_volume(rng, dims, bits)
    vol = pdm.Volume.from_array(vox)
    grid = pdm.BlockGrid.for_dims(dims, b)
    scheme = pdm.scheme_uniform(n, bits)
    pset = pdm.build_pdm_set(vol, grid, scheme, mode)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
    assert np.array_equal(_stack(pset), want)
    mins, maxs = pdm.block_min_max(vol, grid)
    omin, omax = oracle.block_min_max(vox, b)
    assert np.array_equal(mins, omin) and np.array_equal(maxs, omax)
    span = 1 << bits
    for _ in range(3):
        support = np.zeros(span, bool)
        lo = int(rng.integers(0, span))
        support[lo: lo + int(rng.integers(1, span // 3))] = True
        lut = lut_from_support(support, rng)
        tf = pdm.TransferFunction(lut=lut)
        sel = pdm.select_partitions(tf, scheme)
        assert sel.sorted == oracle.select(lut[:, 3], scheme.bounds())
        assert np.array_equal(pdm.combine(pset, sel).dist, oracle.combine(want, sel.sorted))
        assert np.array_equal(pdm.standard_distance_map(vol, grid, tf, mode).dist,
                              oracle.standard_distance_map(vox, b, lut, mode))


def test_device_born_volume_matches_oracle_synth():
    from paper_2407_21552_b200 import synth

    dims, bits = (40, 24, 64), 16
    vol = synth.synth_volume_device(dims, bits, seed=11, nbox=8)
    host = oracle.synth_volume(bits, dims, synth.synth_boxes(dims, bits, 11, 8), seed=11)
    assert np.array_equal(vol.voxels, host)
    assert vol.intensity_range == (int(host.min()), int(host.max()))
    part = synth.synth_volume_device(dims, bits, seed=11, nbox=8, x_range=(8, 30))
    assert np.array_equal(part.voxels, host[8:30])


# --- nibble-packed merge planes (csrc/packed.cu) ---------------------------------------

@pytest.mark.parametrize("dims,b,bits,n,packs", [
    ((64, 40, 64), 4, 16, 32, True),    # z rows of 16 blocks
    ((40, 36, 48), 4, 8, 12, True),     # rows of 12: chunks straddle rows, still <= 11 apart
    ((3, 5, 16), 1, 8, 4, True),        # 240 blocks: last 32-block item is partial
    ((9, 7, 40), 1, 8, 6, None),        # rows of 40: straddling chunks may span > 15
])
def test_packed_merge_matches_oracle(monkeypatch, dims, b, bits, n, packs):
    monkeypatch.setenv("PDM_PACKED", "1")
    rng = np.random.default_rng(sum(dims) * n)
    vox = random_structured_volume(rng, dims, bits)
    vol = pdm.Volume.from_array(vox)
    grid = pdm.BlockGrid.for_dims(dims, b)
    scheme = pdm.scheme_uniform(n, bits)
    pset = pdm.build_pdm_set(vol, grid, scheme)
    maps = oracle.build_pdm_set(vox, b, scheme.bounds(), "range_apron")
    if packs is not None:
        assert (pset.packed() is not None) == packs
    for trial in range(24):
        k = int(rng.integers(1, n + 1)) if trial else n
        s = sorted(rng.choice(np.arange(1, n + 1), size=k, replace=False).tolist())
        got = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset(s), n=n))
        assert np.array_equal(got.dist, oracle.combine(maps, s)), (k, s)
        lut = np.zeros((1 << bits, 4))
        for i in s:
            part = scheme.partitions[i - 1]
            lut[part.rho_lo: part.rho_hi + 1, 3] = 0.25
        dev = pdm.update_from_tf(pset, pdm.TransferFunction(lut=lut))
        assert np.array_equal(dev.device().cpu().numpy(), oracle.combine(maps, s)), (k, s)


@pytest.mark.parametrize("n,map_bytes", [
    (200, 4000),   # flags kernel: per-CTA plane pointer table (n <= 256)
    (300, 2600),   # flags kernel: index x pitch path (n > 256)
])
def test_packed_abi_many_planes(n, map_bytes):
    """pdm_pack_pdms + pdm_combine_packed / pdm_combine_flags_packed straight
    through the C ABI on 1-Lipschitz random-walk planes, against numpy."""
    import torch

    from paper_2407_21552_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(n)
    steps = rng.integers(-1, 2, size=(n, map_bytes))
    maps = np.clip(rng.integers(0, 256, size=(n, 1)) + np.cumsum(steps, axis=1), 0, 255)
    maps = maps.astype(np.uint8)
    pitch = -(-map_bytes // 256) * 256
    planes = torch.zeros((n, pitch), dtype=torch.uint8, device="cuda")
    planes[:, :map_bytes] = torch.from_numpy(maps).cuda()
    chunks = int(L.pdm_packed_chunks(map_bytes))
    nib_pitch, base_pitch = -(-chunks * 8 // 256) * 256, -(-chunks // 256) * 256
    nib = torch.empty((n, nib_pitch), dtype=torch.uint8, device="cuda")
    base = torch.empty((n, base_pitch), dtype=torch.uint8, device="cuda")
    bad = torch.empty(1, dtype=torch.int32, device="cuda")
    st = _lib.stream_handle()
    _lib.check(L.pdm_pack_pdms(_lib.ptr(planes), pitch, map_bytes, n, _lib.ptr(nib), nib_pitch,
                               _lib.ptr(base), base_pitch, _lib.ptr(bad), st), "pack")
    assert int(bad.cpu()[0]) == 0
    tiles = -(-map_bytes // 1024)
    tb = torch.empty((tiles, n), dtype=torch.int16, device="cuda")
    _lib.check(L.pdm_packed_tile_bounds(_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                                        map_bytes, n, _lib.ptr(tb), st), "tile bounds")
    tbh = tb.cpu().numpy().view(np.uint16)
    for t in range(tiles):  # min | max << 8 of each plane over the tile
        seg = maps[:, 1024 * t: 1024 * (t + 1)]
        assert np.array_equal(tbh[t] & 0xFF, seg.min(axis=1))
        assert np.array_equal(tbh[t] >> 8, seg.max(axis=1))
    out = torch.empty(map_bytes, dtype=torch.uint8, device="cuda")
    for k in (1, 7, 33, 64, min(n, 240), n):
        sel = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)
        want = maps[sel].min(axis=0)
        flags = torch.zeros(n, dtype=torch.uint8, device="cuda")
        flags[torch.from_numpy(sel).long().cuda()] = 1
        for tbp in (None, _lib.ptr(tb)):  # without / with the per-tile plane skip
            out.fill_(7)
            _lib.check(L.pdm_combine_flags_packed(_lib.ptr(nib), nib_pitch, _lib.ptr(base),
                                                  base_pitch, tbp, map_bytes, n, _lib.ptr(flags),
                                                  _lib.ptr(out), None, st), "flags")
            assert np.array_equal(out.cpu().numpy(), want), (k, tbp)
            if k <= 240:  # host index list (kernel parameter) path
                out.fill_(7)
                _lib.check(L.pdm_combine_packed(_lib.ptr(nib), nib_pitch, _lib.ptr(base),
                                                base_pitch, tbp, map_bytes, n, sel.ctypes.data, k,
                                                _lib.ptr(out), None, st), "sel")
                assert np.array_equal(out.cpu().numpy(), want), (k, tbp)


@pytest.mark.parametrize("fmt", [1, 2, 3])
def test_merge_packed_to_host_formats_and_pieces(fmt):
    """pdm_merge_packed_to_host through the C ABI: nibble, delta and sparse
    delta forms, 1-7 pieces (piece edges inside and between warp regions),
    device-flag and host-index selections, on 1-Lipschitz planes mixing zero
    plateaus, flat runs and slopes; map sizes with a partial last chunk."""
    import torch

    from paper_2407_21552_b200 import _lib

    L = _lib.lib()
    n = 12
    rng = np.random.default_rng(fmt)
    for map_bytes in (70000, 4096 * 3 + 5):
        steps = rng.choice([-1, 0, 0, 0, 1], size=(n, map_bytes))
        steps[:, rng.integers(0, map_bytes, 40)] = 0
        maps = np.clip(rng.integers(0, 40, size=(n, 1)) + np.cumsum(steps, axis=1), 0, 255)
        maps[:, : map_bytes // 5] = 0  # a zero plateau (all-zero chunks)
        maps = np.clip(maps, 0, 255)
        ok = np.abs(np.diff(maps.astype(np.int16), axis=1)).max() <= 1
        if not ok:  # the plateau edge may jump: make the walk climb out of 0
            maps[:, map_bytes // 5:] = np.minimum(
                maps[:, map_bytes // 5:], np.arange(1, map_bytes - map_bytes // 5 + 1))
        maps = maps.astype(np.uint8)
        pitch = -(-map_bytes // 256) * 256
        planes = torch.zeros((n, pitch), dtype=torch.uint8, device="cuda")
        planes[:, :map_bytes] = torch.from_numpy(maps).cuda()
        chunks = int(L.pdm_packed_chunks(map_bytes))
        nib_pitch, base_pitch = -(-chunks * 8 // 256) * 256, -(-chunks // 256) * 256
        nib = torch.empty((n, nib_pitch), dtype=torch.uint8, device="cuda")
        base = torch.empty((n, base_pitch), dtype=torch.uint8, device="cuda")
        bad = torch.empty(1, dtype=torch.int32, device="cuda")
        st = _lib.stream_handle()
        _lib.check(L.pdm_pack_pdms(_lib.ptr(planes), pitch, map_bytes, n, _lib.ptr(nib),
                                   nib_pitch, _lib.ptr(base), base_pitch, _lib.ptr(bad), st),
                   "pack")
        assert int(bad.cpu()[0]) == 0
        tb = torch.empty((-(-map_bytes // 1024), n), dtype=torch.int16, device="cuda")
        _lib.check(L.pdm_packed_tile_bounds(_lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                                            map_bytes, n, _lib.ptr(tb), st), "tile bounds")
        stage_n = torch.empty(max(chunks * 8, -(-chunks // 64) * 336), dtype=torch.uint8,
                              pin_memory=True)
        stage_b = torch.empty(chunks, dtype=torch.uint8, pin_memory=True)
        for pieces in (1, 3, 7):
            for k in (1, 5, n):
                sel = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)
                want = maps[sel].min(axis=0)
                flags = torch.zeros(n, dtype=torch.uint8, device="cuda")
                flags[torch.from_numpy(sel).long().cuda()] = 1
                for use_flags in (True, False):
                    out = np.full(map_bytes + 32, 0xCD, np.uint8)
                    _lib.check(L.pdm_merge_packed_to_host(
                        _lib.ptr(nib), nib_pitch, _lib.ptr(base), base_pitch,
                        _lib.ptr(tb) if use_flags else None, map_bytes, n,
                        _lib.ptr(flags) if use_flags else None,
                        None if use_flags else sel.ctypes.data, k, stage_n.data_ptr(),
                        stage_b.data_ptr(), out.ctypes.data, pieces, fmt, st), "to_host")
                    assert np.array_equal(out[:map_bytes], want), (map_bytes, pieces, k)
                    assert (out[map_bytes:] == 0xCD).all()


@pytest.mark.parametrize("dims", [
    (48, 32, 64),     # bz = 16: separate packing pass
    (12, 8, 512),     # bz = 128: packing fused into the z pass
    (8, 4, 1024),     # bz = 256: fused
])
def test_packed_planes_decode_to_the_raw_planes(monkeypatch, dims):
    monkeypatch.setenv("PDM_PACKED", "1")
    """Unpack the device's packed planes on the host: base + nibbles == raw."""
    rng = np.random.default_rng(12)
    vox = random_structured_volume(rng, dims, 16)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, 4),
                             pdm.scheme_uniform(8, 16))
    nib, nib_pitch, base, base_pitch = pset.packed()
    nb = pset.grid.num_blocks
    chunks = -(-nb // 32) * 2
    nib = nib.cpu().numpy()[:, :chunks * 8].reshape(8, chunks, 8)
    base = base.cpu().numpy()[:, :chunks]
    vals = np.empty((8, chunks, 16), np.int64)
    vals[:, :, 0::2] = nib & 15
    vals[:, :, 1::2] = nib >> 4
    vals += base[:, :, None]
    raw = np.stack([d.dist.reshape(-1) for d in pset.pdms])
    assert np.array_equal(vals.reshape(8, -1)[:, :nb], raw)
    tiles = -(-nb // 1024)  # + the merge's per-tile plane bounds (uint16 [tiles][n])
    assert pset.device_bytes() == 8 * (pset.plane_pitch + nib_pitch + base_pitch) + 2 * tiles * 8


def test_packed_skipped_for_maps_that_are_not_distance_fields():
    rng = np.random.default_rng(13)
    bdims = (6, 5, 32)
    maps = [rng.integers(0, 256, bdims).astype(np.uint8) for _ in range(5)]
    grid = pdm.BlockGrid.for_dims(bdims, 1)
    pset = pdm.PdmSet(grid=grid, scheme=pdm.scheme_uniform(5, 8),
                      pdms=tuple(pdm.DistanceMap(1, bdims, m) for m in maps))
    s = [1, 3, 4]
    got = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset(s), n=5)).dist
    assert pset.packed() is None
    assert np.array_equal(got, np.minimum.reduce([maps[i - 1] for i in s]))


@pytest.mark.parametrize("fmt", ["3", "2", "1"])
@pytest.mark.parametrize("min_blocks", [0, 1 << 30])
def test_packed_dprime_to_host(monkeypatch, min_blocks, fmt):
    """combine(...).dist over a packable set ships D' packed over PCIe and
    expands it on the host (min_blocks=0 forces that path for these small
    maps; 1 << 30 forces the raw zero-copy path): identical to the oracle
    for device-flag and host-index selections, including a map whose size is
    not a multiple of 16 (rows of 13 blocks still pack: straddling chunks
    stay <= 12 apart)."""
    monkeypatch.setattr(pdm.acceleration, "_HOST_PACKED_MIN_BLOCKS", min_blocks)
    monkeypatch.setenv("PDM_PACKED", "1")
    monkeypatch.setenv("PDM_HOST_FORMAT", fmt)  # delta forms where bz % 16 == 0
    rng = np.random.default_rng(31)
    for dims, b in (((64, 40, 64), 4), ((3, 5, 13), 1)):
        vox = random_structured_volume(rng, dims, 8)
        scheme = pdm.scheme_uniform(8, 8)
        pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, b),
                                 scheme)
        assert pset.packed() is not None
        maps = oracle.build_pdm_set(vox, b, scheme.bounds(), "range_apron")
        for s in ([3], [1, 2, 5, 8], list(range(1, 9))):
            lut = np.zeros((256, 4))
            for i in s:
                part = scheme.partitions[i - 1]
                lut[part.rho_lo: part.rho_hi + 1, 3] = 0.5
            want = oracle.combine(maps, s)
            flags_path = pdm.combine(pset, pdm.select_partitions(pdm.TransferFunction(lut=lut),
                                                                 scheme))
            assert np.array_equal(flags_path.dist, want), (dims, s)
            idx_path = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset(s), n=8))
            assert np.array_equal(idx_path.dist, want), (dims, s)
            assert np.array_equal(idx_path.device().cpu().numpy(), want), (dims, s)


def test_combine_streams_host_view_while_it_is_read(monkeypatch):
    """combine() switches to the one-pass merge that also streams D''s host
    view (pdm_combine_packed_host) only while the caller reads .dist of its
    results, and back when it stops; every result is complete on return and
    equal to the oracle on both sides (HBM and host)."""
    import torch

    monkeypatch.setattr(pdm.acceleration, "_HOST_PACKED_MIN_BLOCKS", 0)
    monkeypatch.setattr(pdm.acceleration, "_HOST_PIECE_ITEMS", 8)  # several pieces
    monkeypatch.setenv("PDM_HOST_FORMAT", "3")
    rng = np.random.default_rng(33)
    dims, b = (64, 48, 128), 2
    vox = random_structured_volume(rng, dims, 8)
    scheme = pdm.scheme_uniform(8, 8)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, b), scheme)
    assert pset.packed() is not None and pset._delta_ok
    maps = oracle.build_pdm_set(vox, b, scheme.bounds(), "range_apron")
    sels = ([2], [1, 3, 8], [4, 5, 6, 7], list(range(1, 9)), [6])
    dual = []
    for i, s in enumerate(sels * 2):
        want = oracle.combine(maps, s)
        dm = pdm.combine(pset, pdm.PartitionSelection(selected=frozenset(s), n=8))
        assert torch.cuda.current_stream().query()
        dual.append(dm._probe.dual)
        assert np.array_equal(dm.device().cpu().numpy(), want), (i, s)
        if i < 7:  # a host reader for the first 7 results, then a device-only one
            assert np.array_equal(dm.dist, want), (i, s)
    assert dual == [False] + [True] * 7 + [False, False]


@pytest.mark.parametrize("dims,b", [
    ((48, 32, 64), 4),      # bz = 16: separate packing pass + pdm_packed_tile_bounds
    ((12, 8, 512), 4),      # bz = 128: bounds taken in the fused z-pass epilogue (8 rows/tile)
    ((9, 6, 1024), 4),      # bz = 256: fused, 4 rows per tile, rows % 4 != 0 at the end
    ((6, 5, 1024), 2),      # bz = 512: fused, 2 rows per tile, odd row count
])
def test_tile_bounds_match_the_planes(monkeypatch, dims, b):
    """The merge's per-tile plane bounds (min | max << 8 over each 1024-block
    tile of every plane), however they were made, equal numpy's over the raw
    planes (partial last tiles included)."""
    monkeypatch.setenv("PDM_PACKED", "1")
    monkeypatch.setenv("PDM_TILE_SKIP", "1")
    rng = np.random.default_rng(17)
    vox = random_structured_volume(rng, dims, 16)
    scheme = pdm.scheme_uniform(8, 16)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, b), scheme)
    assert pset.packed() is not None and pset._tile_bounds is not None
    nb = pset.grid.num_blocks
    raw = np.stack([d.dist.reshape(-1) for d in pset.pdms])
    tb = pset._tile_bounds.cpu().numpy().view(np.uint16)
    for t in range(-(-nb // 1024)):
        seg = raw[:, 1024 * t: 1024 * (t + 1)]
        assert np.array_equal(tb[t] & 0xFF, seg.min(axis=1)), t
        assert np.array_equal(tb[t] >> 8, seg.max(axis=1)), t


def test_packed_disabled_by_env_and_dropped(monkeypatch):
    """PDM_PACKED=0 keeps sets raw; drop_packed() forgets a packed copy; both
    merge paths agree."""
    monkeypatch.setenv("PDM_PACKED", "1")
    rng = np.random.default_rng(41)
    dims = (32, 24, 64)
    vox = random_structured_volume(rng, dims, 16)
    vol, grid, scheme = pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, 4), \
        pdm.scheme_uniform(8, 16)
    packed_set = pdm.build_pdm_set(vol, grid, scheme)
    assert packed_set.packed() is not None
    assert packed_set.device_bytes() > packed_set.n * packed_set.plane_pitch
    monkeypatch.setenv("PDM_PACKED", "0")
    raw_set = pdm.build_pdm_set(vol, grid, scheme)
    assert raw_set.packed() is None
    assert raw_set.device_bytes() == raw_set.n * raw_set.plane_pitch
    sel = pdm.PartitionSelection(selected=frozenset({2, 3, 7}), n=8)
    assert np.array_equal(pdm.combine(raw_set, sel).dist, pdm.combine(packed_set, sel).dist)
    monkeypatch.delenv("PDM_PACKED")
    packed_set.drop_packed()
    assert packed_set._packed is None
    assert np.array_equal(pdm.combine(packed_set, sel).dist, pdm.combine(raw_set, sel).dist)
    assert packed_set.packed() is not None  # re-packed on demand


@pytest.mark.parametrize("packed", [True, False])
def test_merge_writes_stay_inside_the_map(monkeypatch, packed):
    """Guard bytes after D' (map sizes not a multiple of 16 or 32) survive every
    merge path: device flags, host indices, HBM and host destinations."""
    monkeypatch.setenv("PDM_PACKED", "1" if packed else "0")
    rng = np.random.default_rng(51)
    dims = (5, 7, 13)  # 455 blocks
    vox = random_structured_volume(rng, dims, 8)
    scheme = pdm.scheme_uniform(6, 8)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, 1), scheme)
    assert (pset.packed() is not None) == packed
    maps = oracle.build_pdm_set(vox, 1, scheme.bounds(), "range_apron")
    torch = pdm.device.torch()
    nb = pset.grid.num_blocks
    big = torch.full((nb + 64,), 0xAB, dtype=torch.uint8, device="cuda")
    for s in ([2], [1, 3, 6], [1, 2, 3, 4, 5, 6]):
        lut = np.zeros((256, 4))
        for i in s:
            part = scheme.partitions[i - 1]
            lut[part.rho_lo: part.rho_hi + 1, 3] = 0.5
        out = big[:nb].view(pset.grid.bdims)
        pdm.update_from_tf(pset, pdm.TransferFunction(lut=lut), out=out)
        assert np.array_equal(out.cpu().numpy(), oracle.combine(maps, s)), s
        assert int((big[nb:] != 0xAB).sum()) == 0, s
        sel = pdm.PartitionSelection(selected=frozenset(s), n=6)
        host = pdm.combine(pset, sel).dist
        assert np.array_equal(host, oracle.combine(maps, s)), s


@pytest.mark.parametrize("dims,b,bits", [
    ((20, 12, 64), 4, 16),    # apron fast path (16-byte chunks), DT with separate packing
    ((9, 10, 512), 4, 16),    # fused z-pass packing + tile bounds (bz = 128), partial y block
    ((7, 5, 96), 2, 8),       # 8-bit apron fast path, b = 2, partial strip
    ((6, 7, 13), 1, 8),       # generic kernels (nz not a chunk multiple)
    ((8, 1024, 1024), 4, 16),  # TMEM y and z sweeps (256-long lines), fused packing
    ((4, 2048, 2048), 4, 16),  # TMEM y and z sweeps of 512-long lines (16-bit tables)
])
def test_precompute_kernels_write_inside_their_outputs(dims, b, bits):
    """Canary bytes around every precompute output survive (compute-sanitizer
    is closed on this pool; this is the bounds check that replaces it): apron
    min/max and the range_apron mask, the DT planes with the fused packing and
    tile bounds.  Results equal the oracle, so the writes inside are right."""
    import torch

    from paper_2407_21552_b200 import _lib

    L = _lib.lib()
    st = _lib.stream_handle()
    rng = np.random.default_rng(sum(dims) + b)
    vox = random_structured_volume(rng, dims, bits)
    n = 12
    scheme = pdm.scheme_uniform(n, bits)
    grid = pdm.BlockGrid.for_dims(dims, b)
    nb = grid.num_blocks
    vt = pdm.device.to_device(vox)
    G = 256  # canary bytes on each side
    dt = torch.int16 if bits == 16 else torch.uint8
    esz = 2 if bits == 16 else 1

    def guarded(nbytes):
        buf = torch.full((nbytes + 2 * G,), 0xA5, dtype=torch.uint8, device="cuda")
        return buf, buf[G:G + nbytes]

    def intact(buf, nbytes):
        return int((buf[:G] != 0xA5).sum()) == 0 and int((buf[G + nbytes:] != 0xA5).sum()) == 0

    bmn, mn = guarded(nb * esz)
    bmx, mx = guarded(nb * esz)
    _lib.check(L.pdm_block_min_max(_lib.ptr(vt), bits, *dims, b, _lib.ptr(mn), _lib.ptr(mx), st),
               "minmax")
    want_mn, want_mx = oracle.block_min_max(vox, b)
    assert np.array_equal(mn.view(dt).cpu().numpy().view(want_mn.dtype), want_mn.reshape(-1))
    assert np.array_equal(mx.view(dt).cpu().numpy().view(want_mx.dtype), want_mx.reshape(-1))
    assert intact(bmn, nb * esz) and intact(bmx, nb * esz)
    pid = pdm.device.to_device(scheme.pid_lut())
    words = (n + 31) // 32
    bmask, mask = guarded(nb * words * 4)
    _lib.check(L.pdm_partition_mask_range_apron(_lib.ptr(vt), bits, *dims, b, _lib.ptr(pid), n,
                                                _lib.ptr(mask), words, st), "mask")
    assert intact(bmask, nb * words * 4)
    pitch = pdm.device.plane_pitch(nb)
    chunks = int(L.pdm_packed_chunks(nb))
    nib_pitch, base_pitch = -(-chunks * 8 // 256) * 256, -(-chunks // 256) * 256
    tiles = -(-nb // 1024)
    bst, storage = guarded(n * pitch)
    bnib, nib = guarded(n * nib_pitch)
    bbase, base = guarded(n * base_pitch)
    btb, tb = guarded(tiles * n * 2)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(L.pdm_distance_transform_mask_packed(
        _lib.ptr(mask), words, n, *grid.bdims, _lib.ptr(storage), pitch, _lib.ptr(nib), nib_pitch,
        _lib.ptr(base), base_pitch, _lib.ptr(bad), _lib.ptr(tb), st), "dt packed")
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), "range_apron")
    got = storage.view(n, pitch)[:, :nb].cpu().numpy()
    assert np.array_equal(got, np.stack([w.reshape(-1) for w in want]))
    for buf, nbytes in ((bst, n * pitch), (bnib, n * nib_pitch), (bbase, n * base_pitch),
                        (btb, tiles * n * 2)):
        assert intact(buf, nbytes)


def test_merge_fused_zero_count(monkeypatch):
    """combine_flags_into(count_zeros=True): the packed merge counts D''s zero
    blocks itself; occupied_fraction equals the host count (map size not a
    multiple of 32, selections from empty-ish to full)."""
    monkeypatch.setenv("PDM_PACKED", "1")
    rng = np.random.default_rng(61)
    dims = (9, 11, 48)  # 4752 blocks
    vox = random_structured_volume(rng, dims, 8)
    scheme = pdm.scheme_uniform(8, 8)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, 1), scheme)
    assert pset.packed() is not None
    torch = pdm.device.torch()
    for s in ([1], [3, 4], [2, 5, 7], list(range(1, 9))):
        flags = torch.zeros(8, dtype=torch.uint8, device="cuda")
        flags[[i - 1 for i in s]] = 1
        dm = pdm.acceleration.combine_flags_into(pset, flags, count_zeros=True)
        assert dm._zero_count is not None
        want = np.minimum.reduce([pset.pdms[i - 1].dist for i in s])
        assert dm.occupied_fraction == np.count_nonzero(want == 0) / want.size, s
        assert np.array_equal(dm.dist, want), s


@pytest.mark.parametrize("bits", [8, 16])
def test_volume_range_kernel(bits):
    """pdm_volume_range (Volume.intensity_range of a device volume,
    volume.py:86-90): 16-byte vector body, scalar tail, unaligned start; the
    extremes placed in the tail, in the body and at the first voxel."""
    import torch

    from paper_2407_21552_b200 import _lib

    L = _lib.lib()
    dt = np.uint8 if bits == 8 else np.uint16
    top = (1 << bits) - 1
    rng = np.random.default_rng(bits)
    for count in (1, 7, 8, 17, 1000, 4096 + 3, 1 << 20):
        for where in ("body", "tail", "first"):
            h = rng.integers(10, top - 10, count).astype(dt)
            lo_i, hi_i = {"body": (count // 3, count // 2), "tail": (count - 1, count - 2),
                          "first": (0, count // 2)}[where]
            h[hi_i] = top - 3
            h[lo_i] = 2
            for off in (0, 1):  # off 1: the base is not 16-byte aligned
                buf = torch.from_numpy(np.concatenate([np.full(off, 5, dt), h])).cuda()
                src = buf[off:]
                out = torch.empty(2, dtype=torch.int32, device="cuda")
                _lib.check(L.pdm_volume_range(_lib.ptr(src), bits, count, _lib.ptr(out),
                                              _lib.stream_handle()), "range")
                got = tuple(int(v) for v in out.cpu().numpy().view(np.uint32))
                assert got == (int(h.min()), int(h.max())), (count, where, off)


@pytest.mark.parametrize("bits", [8, 16])
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_standard_distance_map_full_and_empty_support(bits, mode):
    """The constant-D shortcut of the full recompute (support = every
    intensity or none) against the oracle, next to a one-intensity-short TF
    that takes the scan + transform path; partial blocks included."""
    rng = np.random.default_rng(bits)
    dims, b = (21, 18, 35), 4
    vox = random_structured_volume(rng, dims, bits)
    vol = pdm.Volume.from_array(vox)
    grid = pdm.BlockGrid.for_dims(dims, b)
    span = 1 << bits
    for fill in ("full", "empty", "all_but_one"):
        lut = np.zeros((span, 4))
        if fill == "full":
            lut[:, 3] = 0.25
        elif fill == "all_but_one":
            lut[:, 3] = 0.25
            lut[int(vox.flat[0]), 3] = 0.0
        got = pdm.standard_distance_map(vol, grid, pdm.TransferFunction(lut=lut), mode).dist
        assert np.array_equal(got, oracle.standard_distance_map(vox, b, lut, mode)), fill


@pytest.mark.parametrize("dims", [(17, 12, 64), (5, 7, 48), (3, 5, 16)])
def test_flags_merge_small_selections_take_the_raw_planes(monkeypatch, dims):
    """pdm_combine_flags_auto: selections of up to pdm_combine_raw_max_k() planes
    merge the raw planes on the device (after the flag compaction), larger ones
    the packed planes; both equal the oracle for k = 0..8, including map sizes
    that leave a byte tail past the last 16-byte chunk."""
    monkeypatch.setenv("PDM_PACKED", "1")
    import torch

    from paper_2407_21552_b200 import _lib

    L = _lib.lib()
    assert L.pdm_combine_raw_max_k() >= 1
    rng = np.random.default_rng(sum(dims))
    vox = random_structured_volume(rng, dims, 8)
    scheme = pdm.scheme_uniform(10, 8)
    pset = pdm.build_pdm_set(pdm.Volume.from_array(vox), pdm.BlockGrid.for_dims(dims, 1), scheme)
    assert pset.packed() is not None
    maps = np.stack([d.dist for d in pset.pdms])
    nb = pset.grid.num_blocks
    nib, nib_pitch, base, base_pitch = pset.packed()
    for k in range(0, 9):
        s = sorted(rng.choice(np.arange(1, 11), size=k, replace=False).tolist())
        flags = torch.zeros(10, dtype=torch.uint8, device="cuda")
        if s:
            flags[[i - 1 for i in s]] = 1
        out = torch.full((nb + 64,), 7, dtype=torch.uint8, device="cuda")
        _lib.check(L.pdm_combine_flags_auto(
            _lib.ptr(pset.storage), pset.plane_pitch, _lib.ptr(nib), nib_pitch, _lib.ptr(base),
            base_pitch, pset.tile_bounds_ptr(), nb, 10, _lib.ptr(flags), _lib.ptr(out), None,
            _lib.stream_handle()), "pdm_combine_flags_auto")
        got = out.cpu().numpy()
        assert np.array_equal(got[:nb].reshape(pset.grid.bdims), oracle.combine(maps, s)), (k, s)
        assert (got[nb:] == 7).all(), k  # nothing written past the map
        dm = pdm.acceleration.combine_flags_into(pset, flags)
        assert np.array_equal(dm.dist, oracle.combine(maps, s)), (k, s)
