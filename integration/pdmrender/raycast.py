"""pdmrender.raycast: the B200 ray marcher (reads D' in HBM, bit-exact with
the reference's float64 marcher); the image-file helpers (save_image,
encode_png: PIL) are taken from the reference module itself."""

from paper_2407_21552_b200.raycast import (  # noqa: F401
    DEFAULT_BLOCK_EDGE,
    ESS_MODES,
    Camera,
    CameraError,
    EssModeError,
    Framebuffer,
    RenderSettings,
    RenderStats,
    camera_rays,
    ess_advance,
    orbit_camera,
    render,
    volume_centre_world,
)
from paper_2407_21552_b200.acceleration import DistanceMap, OccupancyMap  # noqa: F401
from paper_2407_21552_b200.volume import BlockGrid, Volume  # noqa: F401

from . import _refmod

_ref = _refmod.load("raycast")
save_image = _ref.save_image
encode_png = _ref.encode_png
