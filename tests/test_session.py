"""Device-resident TF-edit session (paper_2407_21552_b200.session), the
counterpart of service/session.py:60-127."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2407_21552_b200 as pdm
from conftest import lut_from_support, random_structured_volume
from paper_2407_21552_b200.session import NoSessionError, PdmSessionStore


def test_no_session_errors():
    store = PdmSessionStore()
    with pytest.raises(NoSessionError):
        store.snapshot()
    with pytest.raises(NoSessionError):
        store.set_tf(pdm.tf_archetype("tf2"))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["voxel", "range_apron"])
def test_session_updates_match_oracle(mode):
    rng = np.random.default_rng(21)
    vox = random_structured_volume(rng, (40, 36, 64), 16)
    vol = pdm.Volume.from_array(vox)
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    scheme = pdm.scheme_uniform(16, 16)
    store = PdmSessionStore()
    s0 = store.load(vol, grid, scheme, mode)
    assert np.all(s0.dprime.dist == 255) and len(s0.selection) == 0
    assert s0.dprime_occupied_fraction == 0.0
    pdms = oracle.build_pdm_set(vox, 4, scheme.bounds(), mode)
    held = []
    for _ in range(5):
        support = np.zeros(1 << 16, bool)
        lo = int(rng.integers(0, 1 << 16))
        support[lo: lo + int(rng.integers(1, 20000))] = True
        lut = lut_from_support(support, rng)
        s = store.set_tf(pdm.TransferFunction(lut=lut))
        sel = oracle.select(lut[:, 3], scheme.bounds())
        want = oracle.combine(pdms, sel)
        assert s.selection.sorted == sel
        assert np.isclose(s.dprime_occupied_fraction, np.count_nonzero(want == 0) / want.size)
        assert s.select_ms >= 0 and s.combine_ms > 0
        held.append((s, want))
    for s, want in held:  # earlier snapshots stay valid after later swaps
        assert np.array_equal(s.dprime.dist, want)
    assert store.snapshot() is held[-1][0]
    with pytest.raises(ValueError):
        store.set_tf(pdm.tf_archetype("tf2", bits=8))
