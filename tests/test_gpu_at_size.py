"""Bit-exact parity at the BASELINE.json sizes (configs a-e), on the GPU.

Every check compares the CUDA path with the CPU oracle (oracle/, test
infrastructure) built from the SAME bytes: the shared hash-box generator
(pdm_synth_volume on the device, oracle_synth_volume on the host).

* a: 256^3 u8, b=4, n=8 -- PDM sets (both modes), random 1D TF changes
  (per-intensity random support, conftest.py:34-47), the full recompute.
* b: 512^3 u16, b=8, n=16 -- PDM sets (both modes), merges for random
  intensity-band TFs and aligned TFs, standard_distance_map (both modes).
* c: 1024^3 u16, b=4, n=32 -- PDM sets (both modes), the merge for every
  k = 1..32 (device D' and the host view .dist), the full recompute.
* e: 1024^3 u16, b=4, n=64 -- PDM set and merges for k across 1..64.
* d: 2048^3 u16, b=4, n=32 (2^33 voxels: 64-bit indexing) -- voxel-mode PDM
  set against the oracle built slab by slab (oracle.build_pdm_set_synth), and
  merges at k = 1, 8, 17, 32.

Ref: acceleration.py:184-276, _kernels.py:17-149, transfer.py:250-259.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2407_21552_b200 as pdm

pytestmark = pytest.mark.gpu

SEED = 2407


def _threads():
    oracle.set_threads(oracle.max_threads())


def _device_volume(dims, bits, seed=SEED, nbox=12):
    from paper_2407_21552_b200 import synth

    return synth.synth_volume_device(dims, bits, seed=seed, nbox=nbox)


def _boxes(dims, bits, seed=SEED, nbox=12):
    from paper_2407_21552_b200.synth import synth_boxes

    return synth_boxes(dims, bits, seed, nbox)


def _planes_equal(pset, want) -> None:
    """Every GPU plane == the oracle's, one plane at a time (4.3 GB at d)."""
    nb = pset.grid.num_blocks
    for p in range(pset.n):
        got = pset.storage[p, :nb].cpu().numpy()
        if not np.array_equal(got, want[p].reshape(-1)):
            bad = np.flatnonzero(got != want[p].reshape(-1))
            raise AssertionError(f"plane {p}: {bad.size} blocks differ, first at {bad[0]}")


def _aligned_lut(scheme, picks, rng):
    lut = np.zeros((scheme.intensity_span, 4))
    for p in picks:
        lo, hi = scheme.partitions[p - 1].rho_lo, scheme.partitions[p - 1].rho_hi
        lut[lo: hi + 1, 3] = rng.uniform(0.05, 1.0, hi - lo + 1)
    return lut


def _band_lut(span, rng):
    """1-3 random intensity bands (16-bit random TFs)."""
    lut = np.zeros((span, 4))
    for _ in range(int(rng.integers(1, 4))):
        lo = int(rng.integers(0, span))
        hi = min(span - 1, lo + int(rng.integers(1, span // 6)))
        lut[lo: hi + 1, 3] = rng.uniform(0.05, 1.0, hi - lo + 1)
    return lut


def _check_merges(pset, scheme, want, luts):
    for lut in luts:
        tf = pdm.TransferFunction(lut=lut)
        sel = pdm.select_partitions(tf, scheme)
        wsel = oracle.select(lut[:, 3], scheme.bounds())
        assert sel.sorted == wsel
        wd = oracle.combine(want, wsel)
        dm = pdm.combine(pset, sel)
        assert np.array_equal(dm.device().cpu().numpy(), wd), f"device D' k={len(wsel)}"
        assert np.array_equal(dm.dist, wd), f"host D' k={len(wsel)}"


# --- config a ------------------------------------------------------------------

@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_config_a_256_u8(mode):
    _threads()
    dims, bits, b, n = (256, 256, 256), 8, 4, 8
    vol = _device_volume(dims, bits)
    grid = pdm.BlockGrid.for_dims(dims, b)
    scheme = pdm.scheme_uniform(n, bits)
    vox = oracle.synth_volume(bits, dims, _boxes(dims, bits), SEED)
    assert np.array_equal(vol.device_voxels().cpu().numpy().view(vox.dtype), vox)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
    pset = pdm.build_pdm_set(vol, grid, scheme, mode)
    _planes_equal(pset, want)
    rng = np.random.default_rng(1)
    luts = []
    for p in (0.02, 0.1, 0.5):  # random 1D TF changes (conftest.py:34-47)
        lut = np.zeros((256, 4))
        support = rng.random(256) < p
        lut[support, 3] = rng.uniform(0.05, 1.0, int(support.sum()))
        luts.append(lut)
    _check_merges(pset, scheme, want, luts)
    for lut in luts[:2]:
        got = pdm.standard_distance_map(vol, grid, pdm.TransferFunction(lut=lut), mode).dist
        assert np.array_equal(got, oracle.standard_distance_map(vox, b, lut, mode))


# --- config b ------------------------------------------------------------------

@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_config_b_512_u16(mode):
    _threads()
    dims, bits, b, n = (512, 512, 512), 16, 8, 16
    vol = _device_volume(dims, bits)
    grid = pdm.BlockGrid.for_dims(dims, b)
    scheme = pdm.scheme_uniform(n, bits)
    vox = oracle.synth_volume(bits, dims, _boxes(dims, bits), SEED)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
    pset = pdm.build_pdm_set(vol, grid, scheme, mode)
    _planes_equal(pset, want)
    rng = np.random.default_rng(2)
    luts = [_band_lut(1 << bits, rng) for _ in range(4)]
    luts += [_aligned_lut(scheme, rng.choice(np.arange(1, n + 1), k, replace=False), rng)
             for k in (1, 5, 16)]
    _check_merges(pset, scheme, want, luts)
    minmax = pdm.block_min_max(vol, grid) if mode == "range_apron" else None
    for lut in luts[:3]:
        tf = pdm.TransferFunction(lut=lut)
        wd = oracle.standard_distance_map(vox, b, lut, mode)
        assert np.array_equal(pdm.standard_distance_map(vol, grid, tf, mode).dist, wd)
        if minmax is not None:
            assert np.array_equal(
                pdm.standard_distance_map(vol, grid, tf, mode, minmax=minmax).dist, wd)


# --- configs c and e -------------------------------------------------------------

@pytest.fixture(scope="module")
def config_c_volume():
    _threads()
    dims, bits = (1024, 1024, 1024), 16
    vol = _device_volume(dims, bits)
    vox = oracle.synth_volume(bits, dims, _boxes(dims, bits), SEED)
    return dims, bits, vol, vox


@pytest.mark.parametrize("mode", ["range_apron", "voxel"])
def test_config_c_1024_u16_every_k(config_c_volume, mode):
    dims, bits, vol, vox = config_c_volume
    b, n = 4, 32
    grid = pdm.BlockGrid.for_dims(dims, b)
    scheme = pdm.scheme_uniform(n, bits)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), mode)
    pset = pdm.build_pdm_set(vol, grid, scheme, mode)
    _planes_equal(pset, want)
    rng = np.random.default_rng(3)
    flags = None
    out = None
    for k in range(1, n + 1):  # the config's sweep: every selection size
        picks = sorted(int(i) for i in rng.choice(np.arange(1, n + 1), k, replace=False))
        lut = _aligned_lut(scheme, picks, rng)
        wd = oracle.combine(want, picks)
        # the bench's fused device update (select + merge kernels, caller buffers)
        import torch

        alpha = torch.from_numpy(np.ascontiguousarray(lut[:, 3])).cuda()
        dm = pdm.update_from_tf(pset, alpha, out=out, flags=flags)
        out, flags = dm.device(), None
        assert np.array_equal(out.cpu().numpy(), wd), f"fused update k={k}"
        if k in (1, 2, 7, 16, 31, 32):  # the public API, host view included
            got = pdm.combine(pset, pdm.select_partitions(pdm.TransferFunction(lut=lut), scheme))
            assert np.array_equal(got.dist, wd), f"combine(...).dist k={k}"
    lut = _band_lut(1 << bits, rng)
    tf = pdm.TransferFunction(lut=lut)
    assert np.array_equal(pdm.standard_distance_map(vol, grid, tf, mode).dist,
                          oracle.standard_distance_map(vox, b, lut, mode))


def test_config_e_1024_n64(config_c_volume):
    dims, bits, vol, vox = config_c_volume
    b, n = 4, 64
    grid = pdm.BlockGrid.for_dims(dims, b)
    scheme = pdm.scheme_uniform(n, bits)
    want = oracle.build_pdm_set(vox, b, scheme.bounds(), "range_apron")
    pset = pdm.build_pdm_set(vol, grid, scheme, "range_apron")
    _planes_equal(pset, want)
    rng = np.random.default_rng(5)
    luts = [_aligned_lut(scheme, rng.choice(np.arange(1, n + 1), k, replace=False), rng)
            for k in (1, 9, 33, 64)]
    _check_merges(pset, scheme, want, luts)


# --- config d ------------------------------------------------------------------

def test_config_d_2048_u16_voxel():
    """2^33 voxels on one GPU: PDM set vs the slab-wise oracle, merges."""
    _threads()
    dims, bits, b, n = (2048, 2048, 2048), 16, 4, 32
    scheme = pdm.scheme_uniform(n, bits)
    want = oracle.build_pdm_set_synth(bits, dims, _boxes(dims, bits), SEED, b, scheme.bounds(),
                                      "voxel")
    vol = _device_volume(dims, bits)
    grid = pdm.BlockGrid.for_dims(dims, b)
    pset = pdm.build_pdm_set(vol, grid, scheme, "voxel")
    del vol
    _planes_equal(pset, want)
    rng = np.random.default_rng(4)
    luts = [_aligned_lut(scheme, rng.choice(np.arange(1, n + 1), k, replace=False), rng)
            for k in (1, 8, 17, 32)]
    _check_merges(pset, scheme, want, luts)
