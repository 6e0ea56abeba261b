"""The pdmrender overlay (integration/) binds the reference's callers to the
B200 modules.  Needs /root/reference (this container); no GPU compute."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path(os.environ.get("PDMRENDER_REF", "/root/reference/pkg/src/pdmrender"))

pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference tree not present")

PROBE = r"""
import sys
import pdmrender, paper_2407_21552_b200 as b2
import pdmrender.bench as bench, pdmrender.raycast as raycast, pdmrender.cli as cli
from pdmrender.service import session
assert pdmrender.combine is b2.combine
assert bench.combine is b2.combine and bench.build_pdm_set is b2.build_pdm_set
assert bench.standard_distance_map is b2.standard_distance_map
assert session.combine is b2.combine and session.build_pdm_set is b2.build_pdm_set
assert cli.select_partitions is b2.select_partitions
assert pdmrender.Volume is b2.Volume and pdmrender.BlockGrid is b2.BlockGrid
assert raycast.DistanceMap is b2.DistanceMap
assert raycast.render is b2.render and pdmrender.render is b2.render  # the GPU marcher
assert pdmrender.camera_rays is b2.camera_rays and callable(raycast.encode_png)
assert pdmrender._kernels.__file__.startswith(sys.argv[1])  # non-hot modules stay the reference's
v = pdmrender.synth_volume("two_spheres", 16, seed=1)
assert type(v) is b2.Volume and v.bits == 8
tf = pdmrender.fixture_tf("tf5")
assert type(tf) is b2.TransferFunction
s = pdmrender.scheme_uniform(8, 8)
try:
    pdmrender.combine(pdmrender.PdmSet(grid=pdmrender.BlockGrid.for_dims((8, 8, 8), 4),
                                       scheme=s, pdms=(), occupancy_mode="voxel"),
                      pdmrender.PartitionSelection(selected=frozenset({1}), n=4))
except pdmrender.SelectionError:
    pass
else:
    raise AssertionError("SelectionError expected")
print("overlay ok")
"""


def test_overlay_binds_hot_path():
    env = dict(os.environ, PYTHONPATH=f"{ROOT / 'integration'}:{ROOT}",
               NUMBA_CACHE_DIR="/tmp/numba_cache", PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-c", PROBE, str(REF)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "overlay ok" in r.stdout
