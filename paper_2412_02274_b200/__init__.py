"""B200-native grid-resistance engine (arXiv 2412.02274 hot path) behind the
reference's skypar API.  The compute lives in libskygpu.so (csrc/, sm_100a);
this package is the host-side mirror of the reference interface."""
from .skypar import (  # noqa: F401
    GRES_AUTO, GRES_CELLS, GRES_PAIRS, SKY_AUTO, SKY_GRID, SKY_PARTS, SKY_ROUNDS, GridResistanceResult, PartitionPlan, SkyGpuError,
    SkylineResult, Strategy, assign_partitions, device_count, generate, grid_resistance, make_plan,
    load_dataset_csv, max_grid_intervals, normalize, parallel_skyline, pipeline_csv,
    read_csv_bytes, pipeline, select_representatives, sfs_accounting, skyline_bnl,
    snap_relation, snap_to_grid,
)
