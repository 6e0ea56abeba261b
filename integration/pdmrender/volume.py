"""pdmrender.volume: B200 Volume / BlockGrid / block_min_max; the reference's
non-hot helpers (synth_volume, SYNTH_KINDS) are taken from the reference
module itself, rebound to this module's Volume class."""

from paper_2407_21552_b200.volume import (  # noqa: F401
    BitDepthError,
    BlockGrid,
    SizeMismatchError,
    Volume,
    VolumeError,
    block_min_max,
    load_raw,
    save_raw,
)

from . import _refmod

_ref = _refmod.load("volume")
_ref.Volume = Volume
_ref.VolumeError = VolumeError
synth_volume = _ref.synth_volume
SYNTH_KINDS = _ref.SYNTH_KINDS
