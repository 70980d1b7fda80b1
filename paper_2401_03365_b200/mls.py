"""Python mirror of the MLS projection API (proj/include/pcs/mls.hpp, wls.hpp,
spatial.hpp, parallel.hpp) over the C ABI of include/pcs_lop.h.

Every call runs on the B200 (lib/libpcs_lop_b200.so, mls.cu); there is no CPU
fallback.  Names, parameters, status enums and error behaviour follow the
reference: ``MlsParams.validate`` raises ``InvalidParam`` with the reference's
messages, ``smooth_cloud`` of an empty cloud returns an empty cloud, and a thin
or degenerate neighbourhood degrades the projection instead of failing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Tuple

import numpy as np

from . import _lib as L
from .lop import InvalidParam, KernelParams, _check, _cloud, _ptr


class ProjectionStatus(IntEnum):
    """proj/include/pcs/mls.hpp:32-37."""
    FULL = 0
    DEGRADED_DEGREE = 1
    PLANE_ONLY = 2
    SKIPPED = 3


class PlaneFitStatus(IntEnum):
    """proj/include/pcs/wls.hpp:53-59 (OutOfCoverage is host-side only)."""
    OK = 0
    TOO_FEW_NEIGHBORS = 1
    DEGENERATE_NEIGHBORHOOD = 2
    NO_CONVERGENCE = 3
    OUT_OF_COVERAGE = 4


class PolyFitStatus(IntEnum):
    """proj/include/pcs/wls.hpp:77-82."""
    OK = 0
    TOO_FEW_NEIGHBORS = 1
    SINGULAR_SYSTEM = 2
    OUT_OF_COVERAGE = 3


@dataclass
class MlsParams:
    """proj/include/pcs/mls.hpp:14-30."""
    kernel: KernelParams = field(default_factory=KernelParams)
    degree: int = 2
    plane_tol: float = 1e-10
    plane_max_iter: int = 50

    def validate(self) -> None:
        if not (self.kernel.h > 0.0):
            raise InvalidParam("kernel bandwidth h must be positive")
        if not (self.kernel.cutoff_multiple > 0.0):
            raise InvalidParam("kernel cutoff_multiple must be positive")
        if self.degree < 1 or self.degree > 4:
            raise InvalidParam("MlsParams: degree must be in [1,4]")
        if not (self.plane_tol > 0.0):
            raise InvalidParam("MlsParams: plane_tol must be positive")
        if self.plane_max_iter < 1:
            raise InvalidParam("MlsParams: plane_max_iter must be >= 1")


@dataclass
class MlsResults:
    """Per-query outcome arrays (pcs_mls_result)."""
    projected: np.ndarray      # (m, 3)
    origin: np.ndarray         # (m, 3) plane frame
    normal: np.ndarray
    u: np.ndarray
    v: np.ndarray
    coeffs: np.ndarray         # (m, 15)
    cmin: np.ndarray           # (m, 3) bounds of the query centres used
    cmax: np.ndarray
    status: np.ndarray         # ProjectionStatus
    degree_used: np.ndarray
    iterations: np.ndarray
    plane_status: np.ndarray   # PlaneFitStatus
    poly_status: np.ndarray    # PolyFitStatus


def _desc(params: MlsParams, device: int = -1) -> L.MlsDesc:
    d = L.MlsDesc()
    L.lib().pcs_mls_desc_default(C.byref(d))
    d.h = float(params.kernel.h)
    d.cutoff_multiple = float(params.kernel.cutoff_multiple)
    d.degree = int(params.degree)
    d.plane_tol = float(params.plane_tol)
    d.plane_max_iter = int(params.plane_max_iter)
    d.device = int(device)
    return d


# numpy view of pcs_mls_result (include/pcs_lop.h)
RESULT_DTYPE = np.dtype([("projected", "f8", 3), ("origin", "f8", 3), ("normal", "f8", 3),
                         ("u", "f8", 3), ("v", "f8", 3), ("coeffs", "f8", 15), ("cmin", "f8", 3),
                         ("cmax", "f8", 3), ("status", "i4"), ("degree_used", "i4"),
                         ("iterations", "i4"), ("plane_status", "i4"), ("poly_status", "i4"),
                         ("pad", "i4")])
assert RESULT_DTYPE.itemsize == C.sizeof(L.MlsResultC)


def _results(a: np.ndarray) -> MlsResults:
    return MlsResults(**{k: a[k].copy() for k in RESULT_DTYPE.names if k != "pad"})


def _rptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(L.MlsResultC))


class MlsIndex:
    """A cloud resident on the device (pcs_mls_index): radius queries and
    per-query MLS fits against it (SpatialIndex + wls/mls free functions)."""

    def __init__(self, cloud, device: int = -1):
        self.cloud = _cloud(cloud)
        h = C.c_void_p()
        _check(L.lib().pcs_mls_index_create(_ptr(self.cloud), self.cloud.shape[0], int(device),
                                            C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            L.lib().pcs_mls_index_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def radius_query_all(self, centers, r: float) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """CSR (offsets[m+1], idx, dist) of SpatialIndex::radius_query for every centre
        (proj/src/spatial.cpp:82-111): ascending index per centre, reference distances."""
        Q = _cloud(centers)
        m = Q.shape[0]
        off = np.zeros(m + 1, dtype=np.uint64)
        _check(L.lib().pcs_mls_index_radius(self._h, _ptr(Q), m, float(r), _ptr(off, L._u64p),
                                            None, None, 0))
        tot = int(off[-1])
        idx = np.zeros(max(tot, 1), dtype=np.uint32)
        if tot:
            _check(L.lib().pcs_mls_index_radius(self._h, _ptr(Q), m, float(r), _ptr(off, L._u64p),
                                                _ptr(idx, L._u32p), None, tot))
        idx = idx[:tot]
        out_idx = np.empty_like(idx)
        dist = np.empty(tot, dtype=np.float64)
        for i in range(m):
            a, b = int(off[i]), int(off[i + 1])
            s = np.sort(idx[a:b])
            out_idx[a:b] = s
            d = self.cloud[s] - Q[i]
            dist[a:b] = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
        return off, out_idx, dist

    def project(self, queries, params: MlsParams, mode: int = L.PCS_MLS_PROJECT,
                frames: Optional[np.ndarray] = None, device: int = -1) -> MlsResults:
        """project_point / fit_reference_plane / fit_local_polynomial (mode) for
        every query, one device launch."""
        params.validate()
        Q = _cloud(queries)
        m = Q.shape[0]
        out = np.zeros(max(m, 1), dtype=RESULT_DTYPE)
        fr = None
        if mode == L.PCS_MLS_POLY:
            fr = np.ascontiguousarray(frames, dtype=np.float64).reshape(m, 12)
        d = _desc(params, device)
        _check(L.lib().pcs_mls_project(self._h, C.byref(d), _ptr(Q), m, int(mode),
                                       _ptr(fr) if fr is not None else None, _rptr(out), None))
        return _results(out[:m])


# pcs_mls_outcome: ProjectionOutcome without the point (proj/include/pcs/mls.hpp:38-44)
OUTCOME_DTYPE = np.dtype([("status", "i1"), ("degree_used", "i1"), ("plane_status", "i1"),
                          ("poly_status", "i1"), ("iterations", "i4")])
assert OUTCOME_DTYPE.itemsize == 8


def smooth_cloud(cloud, params: MlsParams, device: int = -1, full_records: bool = False,
                 center_bounds: bool = False) -> Tuple[np.ndarray, MlsResults]:
    """smooth_cloud (proj/src/mls.cpp:75-93): every point projected against the
    untouched input cloud, one device launch; output order = input order.

    As the reference, the call returns the projected cloud and the per-point
    outcome (status, degree used, plane-fit iterations and status); the frames,
    coefficients and centre bounds of ``MlsResults`` are filled only with
    ``full_records=True`` (312 instead of 32 bytes per point cross PCIe);
    ``center_bounds=True`` adds ``cmin`` / ``cmax`` (the bounds of the query
    centres each projection used: what parallel_smooth's coverage test reads)."""
    params.validate()
    P = _cloud(cloud)
    n = P.shape[0]
    out = np.zeros((n, 3), dtype=np.float64)
    if full_records:
        res = np.zeros(max(n, 1), dtype=RESULT_DTYPE)
        if n:
            d = _desc(params, device)
            _check(L.lib().pcs_mls_smooth(C.byref(d), _ptr(P), n, _ptr(out), _rptr(res)))
        return out, _results(res[:n])
    oc = np.zeros(max(n, 1), dtype=OUTCOME_DTYPE)
    oc["status"] = 3  # Skipped
    cb = np.zeros((max(n, 1), 6), dtype=np.float64) if center_bounds else None
    if n:
        d = _desc(params, device)
        if center_bounds:
            _check(L.lib().pcs_mls_smooth_bounds(C.byref(d), _ptr(P), n, _ptr(out),
                                                 oc.ctypes.data_as(C.c_void_p), _ptr(cb)))
        else:
            _check(L.lib().pcs_mls_smooth_outcomes(C.byref(d), _ptr(P), n, _ptr(out),
                                                   oc.ctypes.data_as(C.c_void_p)))
    oc = oc[:n]
    i4 = lambda k: oc[k].astype(np.int32)  # noqa: E731
    return out, MlsResults(projected=out, origin=None, normal=None, u=None, v=None, coeffs=None,
                           cmin=cb[:n, :3].copy() if center_bounds else None,
                           cmax=cb[:n, 3:].copy() if center_bounds else None, status=i4("status"),
                           degree_used=i4("degree_used"), iterations=i4("iterations"),
                           plane_status=i4("plane_status"), poly_status=i4("poly_status"))


def partition(cloud, workers: int, support: float) -> Tuple[int, np.ndarray, np.ndarray]:
    """partition (proj/src/parallel.cpp:64-127), host only: (axis, cuts[W-1],
    worker_of[n])."""
    P = _cloud(cloud)
    n = P.shape[0]
    cuts = np.zeros(max(int(workers) - 1, 1), dtype=np.float64)
    wof = np.zeros(max(n, 1), dtype=np.uint32)
    axis = C.c_int32(0)
    _check(L.lib().pcs_mls_partition(_ptr(P), n, int(workers), float(support), C.byref(axis),
                                     _ptr(cuts), _ptr(wof, L._u32p)))
    return int(axis.value), cuts[: max(int(workers) - 1, 0)], wof[:n]
