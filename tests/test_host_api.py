"""Host-side logic of the drop-in API (CPU only): geometry, schemes, TF
validation, selection/error paths that are raised before any launch, RAW I/O,
the C-ABI library's exports, and the no-CPU-fallback guarantee."""

from __future__ import annotations

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2407_21552_b200 as pdm
from paper_2407_21552_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


# --- C ABI -------------------------------------------------------------------------

def _header_symbols() -> set[str]:
    text = (ROOT / "include" / "pdm_b200.h").read_text()
    return set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(pdm_\w+)\s*\(", text, re.M))


def test_library_exports_every_header_symbol():
    L = _lib.load_library()
    declared = _header_symbols()
    assert declared, "no declarations parsed from include/pdm_b200.h"
    assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name
    assert L.pdm_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    L = _lib.load_library()
    # null pointers / sizes are validated before any CUDA call
    assert L.pdm_combine(None, 16, 16, 1, None, 1, None, None) == _lib.PDM_EINVAL
    assert b"null" in L.pdm_last_error()
    assert L.pdm_select(None, 0, 1, None, 0, 0, None, None) == _lib.PDM_EINVAL
    assert L.pdm_block_min_max(ctypes.c_void_p(16), 12, 4, 4, 4, 4, ctypes.c_void_p(16),
                               ctypes.c_void_p(16), None) == _lib.PDM_EINVAL
    assert b"bits" in L.pdm_last_error()


def test_unpack_packed_host_matches_numpy_decode():
    """pdm_unpack_packed_host (host code, no GPU) against a numpy decode of
    the packed encoding: base per 16-block chunk + 4-bit offsets, block
    16c+2j in the low nibble of byte j; map sizes with a partial last chunk."""
    L = _lib.load_library()
    rng = np.random.default_rng(21)
    for nb in (1, 15, 16, 17, 240, 1000, 4096 + 7):
        chunks = 2 * (-(-nb // 32))
        nib = rng.integers(0, 256, chunks * 8, dtype=np.uint8)
        base = rng.integers(0, 241, chunks, dtype=np.uint8)
        vals = np.empty((chunks, 16), np.int64)
        vals[:, 0::2] = nib.reshape(chunks, 8) & 15
        vals[:, 1::2] = nib.reshape(chunks, 8) >> 4
        want = (vals + base[:, None].astype(np.int64)).reshape(-1)[:nb].astype(np.uint8)
        out = np.zeros(nb, np.uint8)
        assert L.pdm_unpack_packed_host(nib.ctypes.data, base.ctypes.data, nb,
                                        out.ctypes.data) == _lib.PDM_OK
        assert np.array_equal(out, want), nb


def test_library_is_sm100a_only():
    lib = ROOT / "paper_2407_21552_b200" / "lib" / "libpdm_b200.so"
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, out.stdout


def test_no_cpu_fallback(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    vol = pdm.Volume.from_array(np.zeros((8, 8, 8), dtype=np.uint8))
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pdm.build_pdm_set(vol, grid, pdm.scheme_uniform(2, 8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pdm.select_partitions(pdm.tf_archetype("tf2"), pdm.scheme_uniform(4, 8))


# --- geometry / volume ----------------------------------------------------------------

def test_block_grid_ceil_division():
    g = pdm.BlockGrid.for_dims((10, 8, 5), 4)
    assert g.bdims == (3, 2, 2) and g.num_blocks == 12
    assert g.block_of((9, 4, 0)) == (2, 1, 0)
    with pytest.raises(ValueError):
        pdm.BlockGrid.for_dims((8, 8, 8), 0)
    with pytest.raises(ValueError):
        pdm.BlockGrid.for_dims((8, 0, 8), 2)


@pytest.mark.parametrize("dims", [(8, 8, 8), (9, 13, 4), (1, 1, 1), (17, 3, 100)])
@pytest.mark.parametrize("b", [1, 2, 4, 7])
def test_block_grid_bounds(dims, b):
    g = pdm.BlockGrid.for_dims(dims, b)
    for d, bd in zip(dims, g.bdims):
        assert bd * b >= d > (bd - 1) * b


def test_volume_validation():
    with pytest.raises(pdm.BitDepthError):
        pdm.Volume.from_array(np.zeros((2, 2, 2), dtype=np.int32))
    with pytest.raises(pdm.VolumeError):
        pdm.Volume(dims=(2, 2, 3), voxels=np.zeros((2, 2, 2), dtype=np.uint8))
    with pytest.raises(pdm.VolumeError):
        pdm.Volume.from_array(np.zeros((2, 2, 2), dtype=np.uint8), spacing=(1, 0, 1))
    v = pdm.Volume.from_array(np.array([[[3, 9]]], dtype=np.uint16))
    assert v.intensity_range == (3, 9) and v.bits == 16 and v.num_voxels == 2


def _write_raw(tmp_path, payload: bytes, meta: dict):
    d, m = tmp_path / "v.raw", tmp_path / "v.json"
    d.write_bytes(payload)
    m.write_text(json.dumps(meta))
    return d, m


def test_load_raw_layout_and_errors(tmp_path):
    d, m = _write_raw(tmp_path, bytes(range(8)), {"dims": [2, 2, 2], "bits": 8})
    v = pdm.load_raw(d, m)
    assert v.voxels[1, 0, 0] == 1 and v.voxels[0, 1, 0] == 2 and v.voxels[0, 0, 1] == 4
    d, m = _write_raw(tmp_path, np.array([300, 7, 0, 65535], ">u2").tobytes(),
                      {"dims": [4, 1, 1], "bits": 16, "endianness": "be"})
    assert pdm.load_raw(d, m).voxels[:, 0, 0].tolist() == [300, 7, 0, 65535]
    d, m = _write_raw(tmp_path, bytes(10), {"dims": [2, 2, 2], "bits": 8})
    with pytest.raises(pdm.SizeMismatchError):
        pdm.load_raw(d, m)
    d, m = _write_raw(tmp_path, bytes(8), {"dims": [2, 2, 2], "bits": 12})
    with pytest.raises(pdm.BitDepthError):
        pdm.load_raw(d, m)
    d, m = _write_raw(tmp_path, bytes(8), {"dims": [2, 2, 2]})
    with pytest.raises(pdm.VolumeError):
        pdm.load_raw(d, m)


def test_raw_round_trip(tmp_path):
    rng = np.random.default_rng(11)
    for bits, dt in ((8, np.uint8), (16, np.uint16)):
        v = pdm.Volume.from_array(rng.integers(0, 1 << bits, (5, 6, 7)).astype(dt), (1, 2, .5))
        pdm.save_raw(v, tmp_path / "a.raw", tmp_path / "a.json")
        back = pdm.load_raw(tmp_path / "a.raw", tmp_path / "a.json")
        assert np.array_equal(back.voxels, v.voxels) and back.spacing == v.spacing


# --- schemes / TFs / selection errors ---------------------------------------------------

def test_scheme_uniform_and_min_special():
    s = pdm.scheme_uniform(3, 2)  # span 4 -> widths 2,1,1
    assert s.bounds() == [(0, 1), (2, 2), (3, 3)]
    assert pdm.scheme_uniform(4, 8).bounds()[1] == (64, 127)
    assert s.pid_lut().tolist() == [0, 0, 1, 2]
    assert s.partition_of(2) == 2
    m = pdm.scheme_with_min_special(4, 8, 10)
    assert m.bounds()[0] == (0, 10) and m.intensity_span == 256
    with pytest.raises(pdm.SchemeError):
        pdm.scheme_with_min_special(4, 8, 253)
    with pytest.raises(pdm.SchemeError):
        pdm.scheme_uniform(257, 8)
    with pytest.raises(pdm.SchemeError):
        pdm.PartitionScheme((pdm.Partition(0, 3), pdm.Partition(5, 7)))
    with pytest.raises(pdm.SchemeError):
        pdm.PartitionScheme((pdm.Partition(0, 5),))


def test_scheme_matches_oracle_pid_lut():
    import oracle

    for n in (1, 7, 32, 100):
        s = pdm.scheme_uniform(n, 16)
        assert np.array_equal(s.pid_lut(), oracle.pid_lut(s.bounds()))


def test_tf_validation_and_archetypes():
    with pytest.raises(pdm.TransferFunctionError):
        pdm.TransferFunction(lut=np.zeros((255, 4)))
    with pytest.raises(pdm.TransferFunctionError):
        pdm.TransferFunction(lut=np.full((256, 4), 1.5))
    nan = np.zeros((256, 4))
    nan[3, 3] = np.nan
    pdm.TransferFunction(lut=nan)  # NaN passes validation like the reference
    t3 = pdm.tf_archetype("tf3")
    assert t3.nonzero_support().tolist() == list(range(128, 256))
    t4 = pdm.tf_archetype("tf4", bits=4)
    assert t4.nonzero_support().tolist() == [4, 5, 6, 7, 12, 13, 14, 15]
    baked = pdm.bake_lut([(0, 0, 0, 0, 0), (255, 1, 1, 1, 1)], bits=8)
    assert baked.lut[255, 3] == 1.0 and baked.lut[0, 3] == 0.0
    assert pdm.tf_from_json(pdm.tf_to_json(baked)).lut.tolist() == baked.lut.tolist()


def test_selection_errors_raised_before_launch():
    s = pdm.scheme_uniform(4, 8)
    with pytest.raises(pdm.SelectionError):
        pdm.PartitionSelection(selected=frozenset({0}), n=4)
    with pytest.raises(pdm.SelectionError):
        pdm.PartitionSelection(selected=frozenset({5}), n=4)
    tf4bit = pdm.bake_lut([(0, 0, 0, 0, 0), (15, 0, 0, 0, 1)], bits=4)
    with pytest.raises(pdm.SelectionError):
        pdm.select_partitions(tf4bit, s)


def test_combine_and_mode_errors_raised_before_launch():
    grid = pdm.BlockGrid.for_dims((8, 8, 8), 4)
    pset = pdm.PdmSet(grid=grid, scheme=pdm.scheme_uniform(2, 8), pdms=(), occupancy_mode="voxel")
    with pytest.raises(pdm.SelectionError):
        pdm.combine(pset, pdm.PartitionSelection(selected=frozenset({1}), n=4))
    vol = pdm.Volume.from_array(np.zeros((8, 8, 8), dtype=np.uint8))
    with pytest.raises(pdm.OccupancyModeError):
        pdm.occupancy_for_partition(vol, grid, pdm.Partition(0, 1), "apron")
    with pytest.raises(pdm.OccupancyModeError):
        pdm.build_pdm_set(vol, grid, pdm.scheme_uniform(2, 8), "apron")
    with pytest.raises(pdm.VolumeError):
        pdm.build_pdm_set(pdm.Volume.from_array(np.zeros((8, 8, 8), np.uint16)), grid,
                          pdm.scheme_uniform(4, 8))
    with pytest.raises(pdm.VolumeError):
        pdm.occupancy_for_tf(pdm.Volume.from_array(np.zeros((8, 8, 8), np.uint16)), grid,
                             pdm.tf_archetype("tf2", bits=8))
    with pytest.raises(pdm.VolumeError):
        pdm.occupancy_for_tf(vol, pdm.BlockGrid.for_dims((8, 8, 4), 4), pdm.tf_archetype("tf2"))


def test_memory_accounting_and_pitch():
    grid = pdm.BlockGrid.for_dims((16, 16, 16), 4)
    pset = pdm.PdmSet(grid=grid, scheme=pdm.scheme_uniform(16, 8),
                      pdms=tuple(pdm.DistanceMap(4, grid.bdims, np.zeros(grid.bdims, np.uint8))
                                 for _ in range(16)), occupancy_mode="voxel")
    assert pset.memory_bytes() == 16 * grid.num_blocks
    assert pset.plane_pitch % 256 == 0 and pset.plane_pitch >= grid.num_blocks


def test_host_maps_keep_reference_types():
    dm = pdm.DistanceMap(b=4, bdims=(2, 2, 2), dist=np.arange(8, dtype=np.uint8).reshape(2, 2, 2))
    assert dm.dist.dtype == np.uint8 and dm.occupied_fraction == 1 / 8
    with pytest.raises(ValueError):
        pdm.DistanceMap(b=4, bdims=(2, 2, 2), dist=np.zeros((2, 2, 2), np.int32))
    with pytest.raises(ValueError):
        pdm.OccupancyMap(b=4, bdims=(2, 2, 3), occupied=np.zeros((2, 2, 2), bool))
    occ = pdm.OccupancyMap(b=4, bdims=(2, 2, 2), occupied=np.eye(2, dtype=bool)[:, :, None]
                           .repeat(2, axis=2))
    assert occ.occupied_fraction == 0.5


def test_distance_map_dump_format(tmp_path):
    dm = pdm.DistanceMap(b=4, bdims=(2, 3, 1), dist=np.arange(6, dtype=np.uint8).reshape(2, 3, 1))
    pdm.save_distance_map(dm, tmp_path / "d.bin")
    raw = (tmp_path / "d.bin").read_bytes()
    assert raw[:4] == b"PDMD" and len(raw) == 20 + 6
    back = pdm.load_distance_map(tmp_path / "d.bin")
    assert back.b == 4 and back.bdims == (2, 3, 1) and np.array_equal(back.dist, dm.dist)
    (tmp_path / "junk.bin").write_bytes(b"NOPE" + bytes(64))
    with pytest.raises(pdm.VolumeError):
        pdm.load_distance_map(tmp_path / "junk.bin")
    with pytest.raises(pdm.VolumeError):
        pdm.load_pdm_set(tmp_path / "junk.bin")


def test_host_buffer_recycles_only_unreferenced_buffers():
    from paper_2407_21552_b200 import device

    import gc

    a = device.host_buffer((3, 7))
    a[:] = 5
    b = device.host_buffer((3, 7))
    assert not np.shares_memory(a, b)  # a is alive: a second buffer
    addrs = {a.ctypes.data, b.ctypes.data}
    view = a[1:]
    del a
    gc.collect()
    c = device.host_buffer((3, 7))
    assert not np.shares_memory(c, view)  # a slice keeps its buffer in use
    assert (view == 5).all()
    addrs.add(c.ctypes.data)
    del view, b, c
    gc.collect()
    d = device.host_buffer((3, 7))
    e = device.host_buffer((3, 7))
    f = device.host_buffer((3, 7))
    assert {d.ctypes.data, e.ctypes.data, f.ctypes.data} == addrs  # released buffers reused
    assert d.shape == (3, 7) and d.dtype == np.uint8 and d.ctypes.data % 64 == 0


@pytest.mark.parametrize("avx512", [True, False])
def test_unpack_delta_host_matches_numpy_decode(monkeypatch, avx512):
    """pdm_unpack_delta_host (host code, no GPU): base = block 16c, blocks
    1..15 of a chunk from 2-bit (step + 1) codes; 1-Lipschitz random walks
    that touch 0 and 255, map sizes with partial chunk groups; the AVX-512
    path (when the CPU has it) and the SSE2 path."""
    if not avx512:
        monkeypatch.setenv("PDM_NO_AVX512", "1")
    L = _lib.load_library()
    rng = np.random.default_rng(22)
    for nb in (1, 15, 16, 17, 64, 65, 240, 1000, 4096 + 7, 1 << 16):
        chunks = 2 * (-(-nb // 32))
        steps = rng.integers(-1, 2, (chunks, 16))
        start = rng.choice([0, 1, 128, 254, 255], chunks)
        vals = np.clip(start[:, None] + np.cumsum(steps, 1) - steps[:, :1], 0, 255)
        d = np.diff(vals, axis=1) + 1                       # blocks 1..15: 0, 1, 2
        codes = (d << (2 * np.arange(15))).sum(1).astype(np.uint32)
        base = vals[:, 0].astype(np.uint8)
        out = np.zeros(nb, np.uint8)
        assert L.pdm_unpack_delta_host(codes.ctypes.data, base.ctypes.data, nb,
                                       out.ctypes.data) == _lib.PDM_OK
        assert np.array_equal(out, vals.reshape(-1)[:nb].astype(np.uint8)), nb


def _sparse_regions(vals: np.ndarray) -> np.ndarray:
    """numpy restatement of the sparse delta encoder (packed.cu store_sparse):
    vals is (chunks, 16) with chunks a multiple of 64; one 336-byte region per
    64 chunks."""
    chunks = vals.shape[0]
    d = np.diff(vals, axis=1) + 1
    codes = (d << (2 * np.arange(15))).sum(1).astype(np.uint32)
    base = vals[:, 0].astype(np.uint8)
    flat = (d == 1).all(axis=1)
    nz = ~(flat & (base == 0))
    regions = np.zeros((chunks // 64, 336), np.uint8)
    for w in range(chunks // 64):
        sl = slice(64 * w, 64 * w + 64)
        words = [int((m.astype(np.uint64) << np.arange(64, dtype=np.uint64)).sum())
                 for m in (nz[sl], ~flat[sl])]  # bit c: chunk c
        regions[w, :16] = np.array(words, dtype=np.uint64).view(np.uint8)
        b = base[sl][nz[sl]]
        regions[w, 16:16 + b.size] = b
        c = codes[sl][~flat[sl]]
        cofs = 16 + (-(-b.size // 4)) * 4
        regions[w, cofs:cofs + 4 * c.size] = c.view(np.uint8)
    return regions


@pytest.mark.parametrize("avx512", [True, False])
def test_unpack_sparse_host_matches_numpy_encoder(monkeypatch, avx512):
    """pdm_unpack_sparse_host (host code, no GPU) against a numpy encoder of
    the sparse delta form: maps mixing all-zero, flat and coded chunks, sizes
    with partial regions and a partial last chunk."""
    if not avx512:
        monkeypatch.setenv("PDM_NO_AVX512", "1")
    L = _lib.load_library()
    rng = np.random.default_rng(23)
    from paper_2407_21552_b200 import device

    for nb in (1, 16, 17, 1000, 1024, 1025, 4096 + 7, 1 << 16):
        chunks = 64 * (-(-nb // 1024))
        for runs in (1, 8):  # runs of 8: whole 4-chunk vectors flat / zero (fast path)
            kind = np.repeat(rng.choice(3, chunks // runs, p=[0.4, 0.3, 0.3]), runs)
            steps = rng.integers(-1, 2, (chunks, 16))             # zero / flat / coded
            steps[kind != 2] = 0
            start = rng.choice([0, 1, 37, 254, 255], chunks)
            start[kind == 0] = 0
            vals = np.clip(start[:, None] + np.cumsum(steps, 1) - steps[:, :1], 0, 255)
            regions = _sparse_regions(vals)
            # unaligned destination (plain stores) and a 64-byte aligned one
            # (non-temporal stores on AVX-512 hosts)
            buf = device.host_buffer((nb + 64 + 16,))
            for out in (buf[1:nb + 17], buf[(-buf.ctypes.data) % 64:][:nb + 16]):
                out[:] = 0xAB
                assert L.pdm_unpack_sparse_host(regions.ctypes.data, nb,
                                                out.ctypes.data) == _lib.PDM_OK
                assert np.array_equal(out[:nb], vals.reshape(-1)[:nb].astype(np.uint8)), nb
                assert (out[nb:] == 0xAB).all(), nb  # nothing written past map_bytes


def test_gather_host_pool_concurrent_callers():
    """pdm_gather_f64_host (host pool, no GPU): strided column gathers of
    several sizes, from 4 host threads at once (ctypes drops the GIL), each
    result exact; the pool serialises jobs and never loses a unit."""
    import threading

    from paper_2407_21552_b200 import _lib

    L = _lib.load_library()
    rng = np.random.default_rng(8)
    errors = []

    def work(seed):
        r = np.random.default_rng(seed)
        for n in (1, 2047, 2048, 2049, 65536, 100003):
            lut = r.random((n, 4))
            out = np.full(n + 1, -1.0)
            assert L.pdm_gather_f64_host(lut.ctypes.data + 24, n, 4, out.ctypes.data) == 0
            if not (np.array_equal(out[:n], lut[:, 3]) and out[n] == -1.0):
                errors.append((seed, n))

    threads = [threading.Thread(target=work, args=(int(rng.integers(1 << 30)),))
               for _ in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
