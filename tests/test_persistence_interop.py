"""PDM-set / distance-map dumps interoperate with the reference's own
save/load (acceleration.py:279-354), both directions.

CPU: the reference writes, this repo parses (host side); this repo writes a
set of host maps, the reference loads it; error cases.  GPU: a reference
dump streamed into device planes (packed at load, PCIe delta form enabled
only for 1-Lipschitz chunks) and a device-resident set dumped for the
reference.  The reference package is imported from baseline/_ref
(tools/stage_reference.sh) or /root/reference; skipped when neither exists.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2407_21552_b200 as pdm
from conftest import random_structured_volume
from paper_2407_21552_b200 import acceleration as acc

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def ref():
    for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "pdmrender").is_dir():
            sys.path.insert(0, str(cand))
            try:
                import pdmrender
            finally:
                sys.path.remove(str(cand))
            if Path(pdmrender.__file__).resolve().is_relative_to(cand.resolve()):
                return pdmrender
    pytest.skip("reference package not available")


def _ref_set(ref, rng, dims=(13, 9, 20), b=3, n=5, mode="voxel"):
    """A reference-built set (the reference's own build_pdm_set, CPU)."""
    vox = random_structured_volume(rng, dims, 8)
    vol = ref.Volume.from_array(vox)
    grid = ref.BlockGrid.for_dims(vol.dims, b)
    return ref.build_pdm_set(vol, grid, ref.scheme_uniform(n, 8), mode)


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_reference_dump_parses_here(ref, tmp_path, mode):
    rs = _ref_set(ref, np.random.default_rng(1), mode=mode)
    path = tmp_path / "ref.pdms"
    ref.save_pdm_set(rs, path)
    grid, scheme, got_mode, maps = acc._read_pdm_set_host(path)
    assert grid.bdims == rs.grid.bdims and grid.dims == rs.grid.dims and grid.b == rs.grid.b
    assert scheme.bounds() == [(p.rho_lo, p.rho_hi) for p in rs.scheme.partitions]
    assert got_mode == mode
    assert np.array_equal(np.asarray(maps), np.stack([d.dist.reshape(-1) for d in rs.pdms]))


@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_dump_written_here_loads_in_reference(ref, tmp_path, mode):
    rs = _ref_set(ref, np.random.default_rng(2), mode=mode)
    grid = pdm.BlockGrid.for_dims(rs.grid.dims, rs.grid.b)
    scheme = pdm.PartitionScheme(tuple(pdm.Partition(p.rho_lo, p.rho_hi)
                                       for p in rs.scheme.partitions))
    mine = pdm.PdmSet(grid=grid, scheme=scheme, occupancy_mode=mode, pdms=tuple(
        pdm.DistanceMap(b=grid.b, bdims=grid.bdims, dist=d.dist.copy()) for d in rs.pdms))
    path = tmp_path / "mine.pdms"
    pdm.save_pdm_set(mine, path)
    back = ref.load_pdm_set(path)
    assert back.occupancy_mode == mode and back.grid == rs.grid
    assert [(p.rho_lo, p.rho_hi) for p in back.scheme.partitions] == scheme.bounds()
    for a, b in zip(back.pdms, rs.pdms):
        assert np.array_equal(a.dist, b.dist)


def test_distance_map_dumps_both_ways(ref, tmp_path):
    rng = np.random.default_rng(3)
    d = rng.integers(0, 256, size=(7, 5, 9), dtype=np.uint8)
    ref.save_distance_map(ref.DistanceMap(b=4, bdims=d.shape, dist=d), tmp_path / "r.pdmd")
    got = pdm.load_distance_map(tmp_path / "r.pdmd")
    assert got.b == 4 and got.bdims == d.shape and np.array_equal(got.dist, d)
    pdm.save_distance_map(pdm.DistanceMap(b=2, bdims=d.shape, dist=d), tmp_path / "m.pdmd")
    back = ref.load_distance_map(tmp_path / "m.pdmd")
    assert back.b == 2 and np.array_equal(back.dist, d)


def test_truncated_dumps_raise_volume_error(ref, tmp_path):
    rs = _ref_set(ref, np.random.default_rng(4))
    path = tmp_path / "t.pdms"
    ref.save_pdm_set(rs, path)
    raw = path.read_bytes()
    path.write_bytes(raw[:-3])
    with pytest.raises(pdm.VolumeError):
        acc._read_pdm_set_host(path)
    path.write_bytes(raw[:30])
    with pytest.raises(pdm.VolumeError):
        acc._read_pdm_set_host(path)
    path.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(pdm.VolumeError):
        acc._read_pdm_set_host(path)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,b,n", [((13, 9, 20), 3, 5), ((64, 40, 128), 2, 7)])
def test_reference_dump_loads_onto_the_device(ref, tmp_path, monkeypatch, dims, b, n):
    monkeypatch.setattr(acc, "_IO_CHUNK", 4096)  # many staging chunks per map
    rs = _ref_set(ref, np.random.default_rng(5), dims=dims, b=b, n=n, mode="range_apron")
    path = tmp_path / "ref.pdms"
    ref.save_pdm_set(rs, path)
    got = pdm.load_pdm_set(path)
    nb = got.grid.num_blocks
    want = np.stack([d.dist.reshape(-1) for d in rs.pdms])
    assert np.array_equal(got.storage[:, :nb].cpu().numpy(), want)
    assert got._packed not in (None, False)  # packed at load
    if got.grid.bdims[2] % 16 == 0:  # chunks inside z rows: distance maps are 1-Lipschitz
        assert got._delta_ok
    for sel in ({1}, {2, 4}, set(range(1, n + 1)), set()):
        s = frozenset(sel)
        mine = pdm.combine(got, pdm.PartitionSelection(selected=s, n=n)).dist
        theirs = ref.combine(rs, ref.PartitionSelection(selected=s, n=n)).dist
        assert np.array_equal(mine, theirs), sel
    # and back: the device set dumped for the reference
    out = tmp_path / "back.pdms"
    pdm.save_pdm_set(got, out)
    assert out.read_bytes() == path.read_bytes()


@pytest.mark.gpu
def test_loaded_non_distance_maps_skip_the_delta_form(tmp_path, monkeypatch):
    """Maps that are not 1-Lipschitz load fine, merge exactly, and never use
    the PCIe delta forms."""
    monkeypatch.setattr(acc, "_HOST_PACKED_MIN_BLOCKS", 1)
    rng = np.random.default_rng(6)
    grid = pdm.BlockGrid.for_dims((64, 16, 64), 1)
    scheme = pdm.scheme_uniform(3, 8)
    maps = np.clip(rng.integers(0, 15, size=(3,) + grid.bdims) + 40, 0, 255).astype(np.uint8)
    host = pdm.PdmSet(grid=grid, scheme=scheme, occupancy_mode="voxel", pdms=tuple(
        pdm.DistanceMap(b=1, bdims=grid.bdims, dist=m) for m in maps))
    pdm.save_pdm_set(host, tmp_path / "x.pdms")
    got = pdm.load_pdm_set(tmp_path / "x.pdms")
    assert not got._delta_ok and acc._host_format(got) == 1
    d = pdm.combine(got, pdm.PartitionSelection(selected=frozenset({1, 3}), n=3)).dist
    assert np.array_equal(d, np.minimum(maps[0], maps[2]))
