"""ctypes binding of lib/libpcs_lop_b200.so (the C ABI in include/pcs_lop.h).

The shared library is built in-tree (``make -C paper_2401_03365_b200``); there
is no Python or CPU fallback for the operator — if the library or an sm_100
device is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCS_LOP_LIB") or os.path.join(PKG_DIR, "lib", "libpcs_lop_b200.so")

PCS_OK = 0
PCS_ERR_INVALID_PARAM = 1
PCS_ERR_EMPTY_CLOUD = 2
PCS_ERR_NUMERICAL = 3
PCS_ERR_CUDA = 4
PCS_ERR_NCCL = 5
PCS_ERR_NO_DEVICE = 6
PCS_ERR_CAPACITY = 7
PCS_ERR_EMPTY_MESH = 8
PCS_ERR_PARSE = 9
PCS_FMT_XYZ = 0
PCS_FMT_PLY_ASCII = 1

PCS_ETA_INV_CUBE = 0
PCS_ETA_NEG_LINEAR = 1
PCS_PREC_FP64 = 0
PCS_PREC_FP32 = 1

# every symbol declared in include/pcs_lop.h (checked by tests/test_abi.py)
EXPORTED = [
    "pcs_lop_desc_default", "pcs_last_error", "pcs_lop_abi_version", "pcs_lop_validate",
    "pcs_lop_run", "pcs_lop_plan_create", "pcs_lop_plan_destroy", "pcs_lop_plan_upload",
    "pcs_nccl_unique_id", "pcs_lop_plan_set_comm", "pcs_lop_plan_reset", "pcs_lop_plan_run",
    "pcs_lop_plan_synchronize", "pcs_lop_plan_last_run_ms", "pcs_lop_plan_download",
    "pcs_lop_plan_launches", "pcs_radius_query_all", "pcs_density_weights", "pcs_grid_sort", "pcs_generate_surface",
    "pcs_add_noise", "pcs_config_sizes", "pcs_generate_config", "pcs_shard_layout",
    "pcs_loopback_group_create", "pcs_loopback_group_destroy", "pcs_lop_plan_set_loopback",
    "pcs_shard_layout_weighted", "pcs_nearest_all", "pcs_deviation", "pcs_deviation_to_mesh",
    "pcs_format_cloud", "pcs_parse_cloud", "pcs_parse_mesh", "pcs_format_double",
    "pcs_format_cloud_alloc", "pcs_free_buffer", "pcs_lop_plan_record_counts",
    "pcs_lop_plan_query_counts", "pcs_trim_device_pool",
    "pcs_mls_desc_default", "pcs_mls_index_create", "pcs_mls_index_destroy", "pcs_mls_index_radius",
    "pcs_mls_project", "pcs_mls_smooth", "pcs_mls_smooth_outcomes", "pcs_mls_smooth_bounds", "pcs_mls_last_device_ms", "pcs_mls_partition", "pcs_lop_plan_set_graphs",
    "pcs_lop_plan_graph_launches", "pcs_lop_plan_set_positions",
]

PCS_MLS_PROJECT = 0
PCS_MLS_PLANE = 1
PCS_MLS_POLY = 2


class LopDesc(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("h", C.c_double),
        ("cutoff_multiple", C.c_double),
        ("mu", C.c_double),
        ("iterations", C.c_int32),
        ("convergence_tol", C.c_double),
        ("eta_kind", C.c_int32),
        ("density_weights", C.c_int32),
        ("precision", C.c_int32),
        ("device", C.c_int32),
        ("lanes_per_point", C.c_int32),
        ("no_graphs", C.c_int32),
        ("reserved", C.c_int32 * 6),
    ]


class MlsDesc(C.Structure):
    """pcs_mls_desc (MlsParams, proj/include/pcs/mls.hpp:14-30, + the device)."""
    _fields_ = [("struct_size", C.c_uint32), ("h", C.c_double), ("cutoff_multiple", C.c_double),
                ("degree", C.c_int32), ("plane_tol", C.c_double), ("plane_max_iter", C.c_int32),
                ("device", C.c_int32)]


class MlsResultC(C.Structure):
    """pcs_mls_result: one query's projection / plane frame / polynomial."""
    _fields_ = [("projected", C.c_double * 3), ("origin", C.c_double * 3),
                ("normal", C.c_double * 3), ("u", C.c_double * 3), ("v", C.c_double * 3),
                ("coeffs", C.c_double * 15), ("cmin", C.c_double * 3), ("cmax", C.c_double * 3),
                ("status", C.c_int32), ("degree_used", C.c_int32), ("iterations", C.c_int32),
                ("plane_status", C.c_int32), ("poly_status", C.c_int32), ("pad", C.c_int32)]


class DeviationReportC(C.Structure):
    """pcs_deviation_report (DeviationReport, proj/include/pcs/metrics.hpp)."""
    _fields_ = [("n", C.c_uint64), ("mean_distance", C.c_double),
                ("std_deviation", C.c_double), ("max_distance", C.c_double)]


class ParseErrorC(C.Structure):
    """pcs_parse_error: line number and reason of a ParseError."""
    _fields_ = [("line", C.c_int64), ("reason", C.c_char * 256)]


class LopSummaryC(C.Structure):
    _fields_ = [
        ("iterations_run", C.c_int32),
        ("converged", C.c_int32),
        ("isolated_events", C.c_uint64),
        ("coincident_pairs", C.c_uint64),
        ("n_isolated", C.c_uint64),
        ("interactions_attr", C.c_uint64),
        ("interactions_rep", C.c_uint64),
        ("density_pairs", C.c_uint64),
        ("careful_points", C.c_uint64),
        ("last_max_disp", C.c_double),
        ("setup_ms", C.c_double),
        ("sweeps_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("sort_ms", C.c_double),
        ("lane_candidates", C.c_uint64),
    ]


_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", PKG_DIR], check=True)


def lib():
    """Loads the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {PKG_DIR}` "
                "(there is no CPU fallback for the B200 LOP operator)")
        L = C.CDLL(LIB_PATH)
        L.pcs_lop_desc_default.argtypes = [C.POINTER(LopDesc)]
        L.pcs_lop_desc_default.restype = None
        L.pcs_last_error.restype = C.c_char_p
        L.pcs_lop_abi_version.restype = C.c_int32
        L.pcs_lop_validate.argtypes = [C.POINTER(LopDesc)]
        L.pcs_lop_run.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, _dp, C.c_uint64, _dp,
                                  C.POINTER(LopSummaryC), _u32p, C.c_uint64]
        L.pcs_lop_plan_create.argtypes = [C.POINTER(LopDesc), C.POINTER(C.c_void_p)]
        L.pcs_lop_plan_destroy.argtypes = [C.c_void_p]
        L.pcs_lop_plan_destroy.restype = None
        L.pcs_lop_plan_upload.argtypes = [C.c_void_p, _dp, C.c_uint64, _dp, C.c_uint64]
        L.pcs_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.pcs_lop_plan_set_comm.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32]
        L.pcs_loopback_group_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
        L.pcs_loopback_group_destroy.argtypes = [C.c_void_p]
        L.pcs_loopback_group_destroy.restype = None
        L.pcs_lop_plan_set_loopback.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.pcs_lop_plan_reset.argtypes = [C.c_void_p]
        L.pcs_lop_plan_run.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.pcs_lop_plan_synchronize.argtypes = [C.c_void_p]
        L.pcs_lop_plan_last_run_ms.argtypes = [C.c_void_p, _dp]
        L.pcs_lop_plan_download.argtypes = [C.c_void_p, _dp, C.POINTER(LopSummaryC), _u32p,
                                            C.c_uint64]
        L.pcs_lop_plan_launches.argtypes = [C.c_void_p]
        L.pcs_lop_plan_launches.restype = C.c_uint64
        L.pcs_lop_plan_set_graphs.argtypes = [C.c_void_p, C.c_int32]
        L.pcs_lop_plan_set_positions.argtypes = [C.c_void_p, _dp, C.c_uint64]
        L.pcs_lop_plan_graph_launches.argtypes = [C.c_void_p]
        L.pcs_lop_plan_graph_launches.restype = C.c_uint64
        L.pcs_lop_plan_record_counts.argtypes = [C.c_void_p, C.c_int32]
        L.pcs_lop_plan_query_counts.argtypes = [C.c_void_p, C.POINTER(C.c_int32), _u8p, C.c_uint64]
        L.pcs_trim_device_pool.argtypes = [C.c_int32]
        L.pcs_radius_query_all.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, _dp, C.c_uint64,
                                           C.c_double, _u64p, _u32p, C.c_uint64]
        L.pcs_density_weights.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, _dp]
        L.pcs_grid_sort.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, C.c_double, _u32p, _u32p]
        L.pcs_generate_surface.argtypes = [C.c_int32, C.c_uint64, C.c_uint64, _dp]
        L.pcs_add_noise.argtypes = [_dp, C.c_uint64, C.c_double, C.c_uint64]
        L.pcs_config_sizes.argtypes = [C.c_int32, C.c_double, _u64p, _u64p]
        L.pcs_generate_config.argtypes = [C.c_int32, C.c_double, _dp, _dp]
        L.pcs_shard_layout.argtypes = [_u32p, C.c_uint64, C.c_int32, _u32p, _u32p, _u32p, _u32p]
        L.pcs_shard_layout_weighted.argtypes = [_u32p, C.POINTER(C.c_float), C.c_uint64, C.c_int32,
                                                _u32p, _u32p, _u32p, _u32p]
        L.pcs_nearest_all.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, _dp, C.c_uint64, _u32p,
                                      _dp]
        L.pcs_deviation.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, _dp, C.c_uint64,
                                    C.POINTER(DeviationReportC), _dp]
        L.pcs_deviation_to_mesh.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, _dp, C.c_uint64,
                                            C.POINTER(DeviationReportC), _dp]
        L.pcs_format_cloud.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, C.c_int32, C.c_char_p,
                                       C.c_uint64, _u64p]
        L.pcs_parse_cloud.argtypes = [C.POINTER(LopDesc), C.c_char_p, C.c_uint64, C.c_int32, _dp,
                                      C.c_uint64, _u64p, C.POINTER(ParseErrorC)]
        L.pcs_parse_mesh.argtypes = [C.c_char_p, C.c_uint64, _dp, C.c_uint64, _u64p,
                                     C.POINTER(ParseErrorC)]
        L.pcs_format_cloud_alloc.argtypes = [C.POINTER(LopDesc), _dp, C.c_uint64, C.c_int32,
                                             C.POINTER(C.c_void_p), _u64p]
        L.pcs_free_buffer.argtypes = [C.c_void_p]
        L.pcs_free_buffer.restype = None
        L.pcs_mls_desc_default.argtypes = [C.POINTER(MlsDesc)]
        L.pcs_mls_desc_default.restype = None
        L.pcs_mls_index_create.argtypes = [_dp, C.c_uint64, C.c_int32, C.POINTER(C.c_void_p)]
        L.pcs_mls_index_destroy.argtypes = [C.c_void_p]
        L.pcs_mls_index_destroy.restype = None
        L.pcs_mls_index_radius.argtypes = [C.c_void_p, _dp, C.c_uint64, C.c_double, _u64p, _u32p,
                                           _dp, C.c_uint64]
        L.pcs_mls_project.argtypes = [C.c_void_p, C.POINTER(MlsDesc), _dp, C.c_uint64, C.c_int32,
                                      _dp, C.POINTER(MlsResultC), _dp]
        L.pcs_mls_smooth.argtypes = [C.POINTER(MlsDesc), _dp, C.c_uint64, _dp,
                                     C.POINTER(MlsResultC)]
        L.pcs_mls_smooth_outcomes.argtypes = [C.POINTER(MlsDesc), _dp, C.c_uint64, _dp, C.c_void_p]
        L.pcs_mls_smooth_bounds.argtypes = [C.POINTER(MlsDesc), _dp, C.c_uint64, _dp, C.c_void_p, _dp]
        L.pcs_mls_last_device_ms.argtypes = [_dp, _dp]
        L.pcs_mls_partition.argtypes = [_dp, C.c_uint64, C.c_uint64, C.c_double,
                                        C.POINTER(C.c_int32), _dp, _u32p]
        L.pcs_format_double.argtypes = [C.c_double, C.c_char_p]
        L.pcs_format_double.restype = C.c_int32
        for name in EXPORTED:
            fn = getattr(L, name)
            if name in ("pcs_format_double", "pcs_free_buffer", "pcs_mls_desc_default",
                        "pcs_mls_index_destroy"):
                continue
            if fn.restype is C.c_int:  # default restype -> pcs_status
                fn.restype = C.c_int
        _lib = L
    return _lib


def last_error() -> str:
    return lib().pcs_last_error().decode(errors="replace")
