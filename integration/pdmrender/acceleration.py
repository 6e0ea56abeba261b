"""pdmrender.acceleration -> paper_2407_21552_b200.acceleration (the hot path)."""

from paper_2407_21552_b200.acceleration import (  # noqa: F401
    DIST_CLAMP,
    OCCUPANCY_MODES,
    DistanceMap,
    OccupancyMap,
    OccupancyModeError,
    PdmSet,
    build_pdm_set,
    combine,
    distance_transform,
    load_distance_map,
    load_pdm_set,
    occupancy_for_partition,
    occupancy_for_tf,
    save_distance_map,
    save_pdm_set,
    standard_distance_map,
    update_from_tf,
)
