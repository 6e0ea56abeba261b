"""Golden vectors for the GPU ray marcher by RUNNING
THE REFERENCE.  Run here (the container that has /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_render_golden.py

For each scene it stores the inputs (voxels, spacing, LUT, skip field, camera,
settings) and the reference outputs: camera_rays (origin, dirs), the raw
march_rays results (per-ray f64 rgba and int64 counters) and render()'s
framebuffer + stats.  Reference (/root/reference/pkg/src/pdmrender):
  camera_rays ........ raycast.py:163-200
  render ............. raycast.py:232-283 (march_rays: _kernels.py:206-365,
                       safe_box_exit: _kernels.py:152-203)
  orbit_camera ....... raycast.py:138-160
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import pdmrender as ref  # noqa: E402
from conftest import aligned_tf, random_structured_volume  # noqa: E402
from pdmrender import _kernels, raycast  # noqa: E402

OUT = Path(__file__).resolve().parent / "render"


def scene(name, volume, tf, camera, settings, accel, manifest, lut_kind=None):
    """lut_kind: store only the archetype name + a digest instead of the LUT
    (16-bit LUTs are 2 MB); the test rebuilds it with tf_archetype."""
    dist, b = raycast._distance_field_for(volume, settings, accel)
    origin, dirs = ref.camera_rays(camera, settings.width, settings.height, volume)
    n = dirs.shape[0]
    rgba = np.empty((n, 4), np.float64)
    counters = np.empty((n, 4), np.int64)
    _kernels.march_rays(volume.voxels, np.ascontiguousarray(tf.lut), dist, b,
                        float(settings.step), settings.ert_enabled,
                        float(settings.ert_threshold), origin, dirs, rgba, counters)
    fb, stats = ref.render(volume, tf, camera, settings, accel)
    assert np.array_equal(fb.pixels, (np.clip(rgba, 0, 1) * 255.0).round().astype(np.uint8)
                          .reshape(settings.height, settings.width, 4))
    np.savez_compressed(
        OUT / f"{name}.npz", voxels=volume.voxels, spacing=np.array(volume.spacing),
        lut=tf.lut if lut_kind is None else np.zeros((0, 4)),
        lut_kind="" if lut_kind is None else lut_kind,
        lut_sha=hashlib.sha256(np.ascontiguousarray(tf.lut).tobytes()).hexdigest(),
        dist=dist, b=b,
        eye=np.array(camera.eye), look_at=np.array(camera.look_at), up=np.array(camera.up),
        fov=camera.vertical_fov, orbit=camera.orbit_angle,
        width=settings.width, height=settings.height, step=settings.step,
        ess_mode=settings.ess_mode, ert_enabled=settings.ert_enabled,
        ert_threshold=settings.ert_threshold,
        origin=origin, dirs=dirs, rgba=rgba, counters=counters, pixels=fb.pixels,
        stats=np.array([stats.rays, stats.samples_evaluated, stats.samples_skipped,
                        stats.blocks_skipped, stats.ert_terminations]))
    manifest[name] = {"dims": list(volume.dims), "bits": volume.bits, "mode": settings.ess_mode,
                      "size": [settings.width, settings.height], "step": settings.step,
                      "evaluated": stats.samples_evaluated, "skipped": stats.samples_skipped}


def main():
    OUT.mkdir(exist_ok=True)
    manifest = {}
    # 1. the reference's own golden render (tests/test_raycast.py:390-402)
    shell = ref.synth_volume("sphere_shell", 32, seed=3)
    scene("shell32_golden", shell, ref.tf_archetype("tf3"), ref.orbit_camera(shell, angle=0.7),
          ref.RenderSettings(32, 32, step=1.0), None, manifest)
    # 2. mode equivalence scene (test_raycast.py:215-259): none / block / distance / pdm
    grid = ref.BlockGrid.for_dims(shell.dims, 4)
    scheme = ref.scheme_uniform(16, bits=8)
    tf = aligned_tf(scheme, {9, 10, 13}, np.random.default_rng(0))
    accel = {
        "none": None,
        "block": ref.occupancy_for_tf(shell, grid, tf, "range_apron"),
        "distance": ref.standard_distance_map(shell, grid, tf, "range_apron"),
        "pdm": ref.combine(ref.build_pdm_set(shell, grid, scheme, "range_apron"),
                           ref.select_partitions(tf, scheme)),
    }
    cam = ref.orbit_camera(shell, angle=2.1)
    for mode, acc in accel.items():
        scene(f"shell32_{mode}", shell, tf, cam, ref.RenderSettings(24, 24, step=0.5,
                                                                   ess_mode=mode), acc,
              manifest)
    # 3. uint16 volume, anisotropic spacing, non-square viewport, b=2, ERT off
    rng = np.random.default_rng(7)
    # two_spheres widened to 16 bits (x 257) plus banded boxes: mixes empty
    # space, partial blocks and a full intensity range
    vox = ref.synth_volume("two_spheres", (40, 36, 48), seed=5).voxels.astype(np.uint16) * 257
    vox = np.maximum(vox, random_structured_volume(rng, (40, 36, 48), 16).voxels)
    vol16 = ref.Volume.from_array(vox, spacing=(1.0, 1.5, 0.75))
    grid16 = ref.BlockGrid.for_dims(vol16.dims, 2)
    scheme16 = ref.scheme_uniform(8, bits=16)
    tf16 = ref.tf_archetype("tf4", bits=16)
    pdm16 = ref.combine(ref.build_pdm_set(vol16, grid16, scheme16, "range_apron"),
                        ref.select_partitions(tf16, scheme16))
    cam16 = ref.Camera(eye=(-30.0, 55.0, 90.0), look_at=(20.0, 26.0, 17.0), up=(0.0, 0.0, 1.0),
                       vertical_fov=38.0, orbit_angle=5.3)
    for ert in (True, False):
        scene(f"u16_pdm_ert{int(ert)}", vol16, tf16, cam16,
              ref.RenderSettings(20, 12, step=0.7, ess_mode="pdm", ert_enabled=ert,
                                 ert_threshold=0.9), pdm16, manifest, "tf4")
    # camera inside the volume, many orbit turns, distance mode on b=2
    cam_in = ref.Camera(eye=(18.0, 20.0, 30.0), look_at=(2.0, 3.0, 4.0), vertical_fov=100.0,
                        orbit_angle=7 * 2 * np.pi + 0.3)
    scene("u16_inside_distance", vol16, tf16, cam_in,
          ref.RenderSettings(16, 16, step=0.33, ess_mode="distance"),
          ref.standard_distance_map(vol16, grid16, tf16, "voxel"), manifest, "tf4")
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")
    print(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
