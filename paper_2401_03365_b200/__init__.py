"""B200-native LOP/WLOP (drop-in for pcs::lop_project of arXiv 2401.03365's reference).

The operator runs as hand-written sm_100a CUDA kernels in
``lib/libpcs_lop_b200.so`` behind the C ABI of ``include/pcs_lop.h``.
"""
from .lop import (  # noqa: F401
    CONFIGS, DeviationReport, EmptyCloud, EmptyMesh, Error, InvalidParam, KernelParams, LopParams, LopPlan, LopSummary,
    LoopbackGroup,
    NumericalFailure, DeviceUnavailable, add_noise, config_params, config_sizes, density_weights, generate_config,
    generate_surface, grid_sort, lop_project, radius_query_all, shard_layout,
    nearest_all, deviation, deviation_to_mesh, ParseError, format_from_path, format_cloud,
    parse_cloud, read_cloud, write_cloud, parse_mesh, format_double, trim_device_pool,
)
from .mls import (  # noqa: F401
    MlsIndex, MlsParams, MlsResults, PlaneFitStatus, PolyFitStatus, ProjectionStatus, partition,
    smooth_cloud,
)

__all__ = [
    "CONFIGS", "EmptyCloud", "Error", "InvalidParam", "KernelParams", "LopParams", "LopPlan",
    "LoopbackGroup",
    "LopSummary", "NumericalFailure", "DeviceUnavailable", "add_noise", "config_params",
    "config_sizes", "density_weights", "generate_config", "generate_surface", "grid_sort", "lop_project",
    "radius_query_all", "shard_layout", "DeviationReport", "EmptyMesh", "nearest_all",
    "deviation", "deviation_to_mesh", "ParseError", "format_from_path", "format_cloud",
    "parse_cloud", "read_cloud", "write_cloud", "parse_mesh", "format_double", "trim_device_pool",
    "MlsIndex", "MlsParams", "MlsResults", "PlaneFitStatus", "PolyFitStatus", "ProjectionStatus",
    "partition", "smooth_cloud",
]
