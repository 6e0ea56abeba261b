"""GPU consumer of D' (raycast.py / csrc/raycast.cu) against goldens made by
running the reference's renderer (tests/golden/make_render_golden.py):
framebuffers, per-ray float64 rgba and work counters must be bit-identical.
CPU-only tests cover the host camera math and the skip arithmetic."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2407_21552_b200 as pdm
from paper_2407_21552_b200 import raycast

GOLD = Path(__file__).resolve().parent / "golden" / "render"
SCENES = sorted(json.loads((GOLD / "manifest.json").read_text()))


def _load(name):
    g = dict(np.load(GOLD / f"{name}.npz"))
    vol = pdm.Volume.from_array(g["voxels"], spacing=tuple(g["spacing"]))
    kind = str(g["lut_kind"])
    tf = pdm.tf_archetype(kind, bits=vol.bits) if kind else pdm.TransferFunction(lut=g["lut"])
    assert hashlib.sha256(np.ascontiguousarray(tf.lut).tobytes()).hexdigest() == str(g["lut_sha"])
    cam = pdm.Camera(eye=tuple(g["eye"]), look_at=tuple(g["look_at"]), up=tuple(g["up"]),
                     vertical_fov=float(g["fov"]), orbit_angle=float(g["orbit"]))
    settings = pdm.RenderSettings(int(g["width"]), int(g["height"]), step=float(g["step"]),
                                  ess_mode=str(g["ess_mode"]),
                                  ert_enabled=bool(g["ert_enabled"]),
                                  ert_threshold=float(g["ert_threshold"]))
    return g, vol, tf, cam, settings


def _accel(g, settings):
    mode, b, dist = settings.ess_mode, int(g["b"]), g["dist"]
    if mode == "none":
        return None
    if mode == "block":  # the reference's field is where(occupied, 0, 1)
        return pdm.OccupancyMap(b, dist.shape, dist == 0)
    return pdm.DistanceMap(b, dist.shape, dist)


# --- host side (no GPU) -------------------------------------------------------------

@pytest.mark.parametrize("name", SCENES)
def test_camera_rays_host_matches_reference(name):
    g, vol, _, cam, settings = _load(name)
    origin, dirs = pdm.camera_rays(cam, settings.width, settings.height, vol)
    assert np.array_equal(origin, g["origin"])
    assert np.array_equal(dirs, g["dirs"])


@pytest.mark.parametrize("threads", [1, 4])
@pytest.mark.parametrize("name", SCENES)
def test_oracle_marcher_matches_reference(name, threads):
    """The C restatement (oracle/march_oracle.c: the checker and the CPU
    baseline of tools/render_bench.py) is pinned to the same goldens."""
    import oracle

    g, vol, tf, _, settings = _load(name)
    oracle.set_threads(threads)
    try:
        rgba, counters = oracle.march_rays(g["voxels"], tf.lut, g["dist"], int(g["b"]),
                                           settings.step, settings.ert_enabled,
                                           settings.ert_threshold, g["origin"], g["dirs"])
    finally:
        oracle.set_threads(1)
    assert np.array_equal(rgba.view(np.uint64), g["rgba"].view(np.uint64)), name
    assert np.array_equal(counters, g["counters"]), name


def test_camera_and_settings_validation():
    with pytest.raises(pdm.CameraError):
        pdm.Camera(eye=(1.0, 2.0, 3.0), look_at=(1.0, 2.0, 3.0))
    with pytest.raises(pdm.CameraError):
        pdm.Camera(eye=(0.0, 0.0, 0.0), look_at=(0.0, 5.0, 0.0))  # up parallel to view
    for fov in (0.0, 180.0):
        with pytest.raises(pdm.CameraError):
            pdm.Camera(eye=(0.0, 0.0, 0.0), look_at=(1.0, 0.0, 0.0), vertical_fov=fov)
    with pytest.raises(ValueError):
        pdm.RenderSettings(0, 4)
    with pytest.raises(ValueError):
        pdm.RenderSettings(4, 4, step=0.0)
    with pytest.raises(ValueError):
        pdm.RenderSettings(4, 4, ert_threshold=0.0)
    with pytest.raises(pdm.EssModeError):
        pdm.RenderSettings(4, 4, ess_mode="bvh")


class TestEssAdvance:
    """The reference's skip-arithmetic expectations (tests/test_raycast.py:291-358)."""

    GRID = pdm.BlockGrid.for_dims((64, 64, 64), 4)

    def _dm(self, value):
        return pdm.DistanceMap(4, self.GRID.bdims, np.full(self.GRID.bdims, value, np.uint8))

    def test_occupied_and_none_step_once(self):
        ray = ((10.0, 10.0, 10.0), (1.0, 0.0, 0.0))
        assert pdm.ess_advance("distance", self._dm(0), (2, 2, 2), ray, 3.0, self.GRID, 0.0,
                               0.5) == pytest.approx(3.5)
        assert pdm.ess_advance("none", None, (2, 2, 2), ray, 3.0, self.GRID, 0.0,
                               0.5) == pytest.approx(3.5)

    def test_distance_jumps(self):
        ray = ((10.0, 10.0, 10.0), (1.0, 0.0, 0.0))
        # d=1: exit of block 2 at x=12 -> t=2; d=5: blocks [-2, 6] -> x=28 -> t=18
        assert pdm.ess_advance("pdm", self._dm(1), (2, 2, 2), ray, 0.0, self.GRID, 0.0,
                               0.5) == pytest.approx(2.0)
        assert pdm.ess_advance("pdm", self._dm(5), (2, 2, 2), ray, 0.0, self.GRID, 0.0,
                               0.5) == pytest.approx(18.0)

    def test_always_advances_and_stays_on_grid(self):
        ray = ((10.0, 10.0, 10.0), (0.6, 0.0, 0.8))
        t = pdm.ess_advance("pdm", self._dm(3), (2, 2, 2), ray, 7.3, self.GRID, 0.1, 0.7)
        assert t > 7.3
        k = (t - 0.1) / 0.7
        assert abs(k - round(k)) < 1e-9

    def test_type_contract(self):
        ray = ((1.0, 1.0, 1.0), (1.0, 0.0, 0.0))
        with pytest.raises(pdm.EssModeError):
            pdm.ess_advance("bvh", None, (0, 0, 0), ray, 0.0, self.GRID, 0.0, 0.5)
        with pytest.raises(pdm.EssModeError):
            pdm.ess_advance("block", self._dm(0), (0, 0, 0), ray, 0.0, self.GRID, 0.0, 0.5)
        with pytest.raises(ValueError):
            pdm.ess_advance("none", None, (0, 0, 0), ray, 0.0, self.GRID, 0.0, 0.0)


# --- device (B200) ---------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENES)
def test_render_matches_reference_bit_for_bit(name):
    g, vol, tf, cam, settings = _load(name)
    accel = _accel(g, settings)
    fb, stats = pdm.render(vol, tf, cam, settings, accel)
    assert np.array_equal(fb.pixels, g["pixels"]), name
    rays, ev, sk, bl, ert = (int(v) for v in g["stats"])
    assert (stats.rays, stats.samples_evaluated, stats.samples_skipped, stats.blocks_skipped,
            stats.ert_terminations) == (rays, ev, sk, bl, ert)
    # per ray: float64 rgba bit patterns and the four counters
    _, _, rgba, counters = raycast._march(vol, tf, cam, settings, accel, per_ray=True)
    assert np.array_equal(rgba.cpu().numpy().view(np.uint64), g["rgba"].view(np.uint64)), name
    assert np.array_equal(counters.cpu().numpy(), g["counters"]), name


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENES)
def test_device_camera_rays_match_reference(name):
    import torch

    from paper_2407_21552_b200 import _lib

    g, vol, _, cam, settings = _load(name)
    origin, fwd, right, up, tan_half, aspect, sp = raycast._camera_frame(
        cam, settings.width, settings.height, vol)
    n = settings.width * settings.height
    dirs = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    frame = np.ascontiguousarray(np.concatenate([fwd, right, up]))
    spc = np.ascontiguousarray(sp)
    _lib.check(_lib.lib().pdm_camera_rays(frame.ctypes.data, tan_half, aspect, spc.ctypes.data,
                                          settings.width, settings.height, _lib.ptr(dirs),
                                          _lib.stream_handle()), "rays")
    assert np.array_equal(dirs.cpu().numpy().view(np.uint64), g["dirs"].view(np.uint64))


@pytest.mark.gpu
def test_render_consumes_device_dprime_from_this_pipeline():
    """D' built and merged here (device-resident, never copied to the host)
    steers the marcher to the reference's pdm framebuffer."""
    g, vol, tf, cam, settings = _load("shell32_pdm")
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    scheme = pdm.scheme_uniform(16, bits=8)
    dprime = pdm.combine(pdm.build_pdm_set(vol, grid, scheme, "range_apron"),
                         pdm.select_partitions(tf, scheme))
    fb, stats = pdm.render(vol, tf, cam, settings, dprime)
    assert dprime._host is None  # consumed on the device
    assert np.array_equal(fb.pixels, g["pixels"])
    assert stats.samples_evaluated == int(g["stats"][1])
    assert np.array_equal(dprime.dist, g["dist"])


@pytest.mark.gpu
def test_render_contract_errors():
    g, vol, tf, cam, settings = _load("shell32_pdm")
    with pytest.raises(ValueError):  # LUT length must match the volume's bits
        pdm.render(vol, pdm.tf_archetype("tf3", bits=10), cam, settings, _accel(g, settings))
    with pytest.raises(pdm.EssModeError):
        pdm.render(vol, tf, cam, settings, None)
    with pytest.raises(pdm.EssModeError):
        pdm.render(vol, tf, cam, pdm.RenderSettings(8, 8, ess_mode="none"), _accel(g, settings))
    with pytest.raises(pdm.EssModeError):  # block dims must fit the volume
        pdm.render(vol, tf, cam, settings, pdm.DistanceMap(2, (15, 16, 16),
                                                           np.zeros((15, 16, 16), np.uint8)))
