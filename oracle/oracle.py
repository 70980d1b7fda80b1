"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/liborc.so`` (the C restatement, lop_oracle.c) and, when it was
built, ``oracle/_ref/libpcs_ref.so`` (the unmodified reference compiled from
/root/reference by oracle/Makefile).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libpcs_ref.so")
# the same unmodified reference objects with lop.cpp's |eta'| call bound to 1
# (eta = -r; oracle/ref_etar_wrap.cpp, linked with -Wl,--wrap)
REF_ETAR_PATH = os.path.join(HERE, "_ref", "libpcs_ref_etar.so")

ETA_INV_CUBE = 0
ETA_NEG_LINEAR = 1

_c_dbl_p = C.POINTER(C.c_double)
_c_u64_p = C.POINTER(C.c_uint64)
_c_u32_p = C.POINTER(C.c_uint32)
_c_u8_p = C.POINTER(C.c_uint8)


class OrcParams(C.Structure):
    _fields_ = [
        ("h", C.c_double),
        ("cutoff_multiple", C.c_double),
        ("mu", C.c_double),
        ("iterations", C.c_int32),
        ("convergence_tol", C.c_double),
        ("eta_kind", C.c_int32),
        ("density_weights", C.c_int32),
        ("store_f32", C.c_int32),
    ]


class OrcSummary(C.Structure):
    _fields_ = [
        ("iterations_run", C.c_int32),
        ("converged", C.c_int32),
        ("isolated_events", C.c_uint64),
        ("coincident_pairs", C.c_uint64),
        ("n_isolated", C.c_uint64),
        ("interactions_attr", C.c_uint64),
        ("interactions_rep", C.c_uint64),
        ("density_pairs_x", C.c_uint64),
        ("density_pairs_p", C.c_uint64),
        ("last_max_disp", C.c_double),
    ]


class RefSummary(C.Structure):
    _fields_ = [
        ("iterations_run", C.c_int32),
        ("converged", C.c_int32),
        ("isolated_events", C.c_uint64),
        ("coincident_pairs", C.c_uint64),
        ("n_isolated", C.c_uint64),
    ]


@dataclass
class Result:
    points: np.ndarray
    iterations_run: int
    converged: bool
    isolated_events: int
    coincident_pairs: int
    isolated_indices: np.ndarray
    interactions_attr: int = 0
    interactions_rep: int = 0
    last_max_disp: float = 0.0
    flags: np.ndarray = None


def build(reference: bool = True) -> None:
    """Build liborc.so (and _ref when /root/reference is present)."""
    targets = ["oracle"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_orc = None
_ref = None


def _ptr(a, t):
    return a.ctypes.data_as(t)


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_PATH):
            build(reference=False)
        lib = C.CDLL(ORC_PATH)
        lib.orc_lop_project.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                        C.POINTER(OrcParams), _c_dbl_p, C.POINTER(OrcSummary),
                                        _c_u32_p, C.c_int]
        lib.orc_lop_project_flags.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                              C.POINTER(OrcParams), _c_dbl_p,
                                              C.POINTER(OrcSummary), _c_u32_p, _c_u8_p, C.c_int]
        lib.orc_lop_sweep.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                      C.POINTER(OrcParams), _c_dbl_p, _c_u8_p, _c_u32_p,
                                      _c_dbl_p, C.c_int]
        lib.orc_lop_sweep_rows.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                           C.POINTER(OrcParams), _c_u32_p, C.c_size_t, _c_dbl_p,
                                           C.POINTER(C.c_int32), C.c_int]
        lib.orc_radius_query_all.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                             C.c_double, _c_u64_p, _c_u32_p, _c_dbl_p, C.c_int]
        lib.orc_density_weights.argtypes = [_c_dbl_p, C.c_size_t, C.c_double, C.c_double,
                                            _c_dbl_p, C.c_int]
        lib.orc_add_noise.argtypes = [_c_dbl_p, C.c_size_t, C.c_double, C.c_uint64]
        lib.orc_plane.argtypes = [_c_dbl_p, C.c_size_t, C.c_uint64]
        lib.orc_sphere.argtypes = [_c_dbl_p, C.c_size_t, C.c_uint64]
        lib.orc_config_sizes.argtypes = [C.c_int, C.c_double, _c_u64_p, _c_u64_p]
        lib.orc_generate_config.argtypes = [C.c_int, C.c_double, _c_dbl_p, _c_dbl_p]
        lib.orc_theta.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.orc_theta.restype = C.c_double
        lib.orc_nearest_all.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t, _c_u32_p,
                                        _c_dbl_p, C.c_int]
        lib.orc_deviation.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t, _c_dbl_p,
                                      _c_dbl_p, C.c_int]
        lib.orc_point_triangle_distance.argtypes = [_c_dbl_p, _c_dbl_p]
        lib.orc_point_triangle_distance.restype = C.c_double
        lib.orc_deviation_to_mesh.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                              _c_dbl_p, _c_dbl_p, C.c_int]
        lib.orc_mls_project.argtypes = [_c_dbl_p, C.c_size_t, _c_dbl_p, C.c_size_t,
                                        C.POINTER(OrcMlsParams), C.c_int, _c_dbl_p, C.c_void_p,
                                        C.c_int]
        _orc = lib
    return _orc


class OrcMlsParams(C.Structure):
    _fields_ = [("h", C.c_double), ("cutoff", C.c_double), ("degree", C.c_int),
                ("tol", C.c_double), ("max_iter", C.c_int)]


# orc_mls_result (lop_oracle.h)
MLS_DTYPE = np.dtype([("projected", "f8", 3), ("origin", "f8", 3), ("normal", "f8", 3),
                      ("u", "f8", 3), ("v", "f8", 3), ("coeffs", "f8", 15), ("status", "i4"),
                      ("degree_used", "i4"), ("iterations", "i4"), ("plane_status", "i4"),
                      ("poly_status", "i4"), ("pad", "i4")])
MLS_PROJECT, MLS_PLANE, MLS_POLY = 0, 1, 2


def mls_project(C_pts, Q, h, cutoff=3.0, degree=2, tol=1e-10, max_iter=50, mode=MLS_PROJECT,
                frames=None, threads=0) -> np.ndarray:
    """orc_mls_project — the C restatement of project_point / fit_reference_plane /
    fit_local_polynomial (proj/src/mls.cpp:28-69, wls.cpp:53-222) per query;
    returns a structured array (MLS_DTYPE)."""
    Cc = _xyz(C_pts)
    Qq = _xyz(Q)
    m = Qq.shape[0]
    out = np.zeros(max(m, 1), dtype=MLS_DTYPE)
    fr = None
    if mode == MLS_POLY:
        fr = np.ascontiguousarray(frames, dtype=np.float64).reshape(m, 12)
    prm = OrcMlsParams(h, cutoff, degree, tol, max_iter)
    rc = orc().orc_mls_project(_ptr(Cc, _c_dbl_p), Cc.shape[0], _ptr(Qq, _c_dbl_p), m,
                               C.byref(prm), mode, _ptr(fr, _c_dbl_p) if fr is not None else None,
                               out.ctypes.data_as(C.c_void_p), threads)
    if rc:
        raise OracleError(rc)
    return out[:m]


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


_ref_etar = None


def ref(eta: int = ETA_INV_CUBE):
    """The reference build: eta = 1/(3r^3) as the reference ships it, or (eta =
    ETA_NEG_LINEAR) the same objects with |eta'| bound to 1."""
    global _ref, _ref_etar
    if eta == ETA_NEG_LINEAR:
        if _ref_etar is None:
            if not os.path.exists(REF_ETAR_PATH):
                raise FileNotFoundError(REF_ETAR_PATH)
            _ref_etar = _bind_ref(C.CDLL(REF_ETAR_PATH))
        return _ref_etar
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_PATH)
        _ref = _bind_ref(C.CDLL(REF_PATH))
    return _ref


def _bind_ref(lib):
    if True:
        lib.ref_lop_project.argtypes = [_c_dbl_p, C.c_uint64, _c_dbl_p, C.c_uint64, C.c_double,
                                        C.c_double, C.c_double, C.c_int, C.c_double, _c_dbl_p,
                                        C.POINTER(RefSummary), _c_u32_p]
        lib.ref_radius_query_all.argtypes = [_c_dbl_p, C.c_uint64, _c_dbl_p, C.c_uint64,
                                             C.c_double, _c_u64_p, _c_u32_p, _c_dbl_p]
        lib.ref_add_noise.argtypes = [_c_dbl_p, C.c_uint64, C.c_double, C.c_uint64]
        lib.ref_generate_surface.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _c_dbl_p]
        lib.ref_theta.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.ref_theta.restype = C.c_double
        lib.ref_index_build_ms.argtypes = [_c_dbl_p, C.c_uint64]
        lib.ref_index_build_ms.restype = C.c_double
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_nearest_all.argtypes = [_c_dbl_p, C.c_uint64, _c_dbl_p, C.c_uint64, _c_u32_p,
                                        _c_dbl_p, C.c_int]
        lib.ref_deviation.argtypes = [_c_dbl_p, C.c_uint64, _c_dbl_p, C.c_uint64, _c_dbl_p,
                                      _c_dbl_p]
        lib.ref_deviation_to_mesh.argtypes = [_c_dbl_p, C.c_uint64, _c_dbl_p, C.c_uint64,
                                              _c_dbl_p, _c_dbl_p]
        lib.ref_format_cloud.argtypes = [_c_dbl_p, C.c_uint64, C.c_int, C.c_char_p, C.c_uint64,
                                         _c_u64_p]
        lib.ref_parse_cloud.argtypes = [C.c_char_p, C.c_uint64, C.c_int, _c_dbl_p, C.c_uint64,
                                        _c_u64_p, C.POINTER(C.c_int64)]
        lib.ref_point_triangle_distance.argtypes = [_c_dbl_p, _c_dbl_p]
        lib.ref_point_triangle_distance.restype = C.c_double
    return lib


def _xyz(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))
    return a


ERRORS = {1: "InvalidParam", 2: "EmptyCloud", 3: "NoMemory"}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        self.kind = ERRORS.get(code, "Error")
        super().__init__(f"{self.kind}({code}) {what}")


def lop_project(P, X0, h, cutoff=3.0, mu=0.4, iterations=30, tol=1e-7,
                eta=ETA_INV_CUBE, wlop=False, threads=0, store_f32=False,
                flags=False) -> Result:
    """orc_lop_project — the C restatement of pcs::lop_project (+eta/WLOP).
    flags=True also returns per-point event flags (Result.flags, OR over sweeps
    >= 2: 1 isolated, 2 anchored, 8 a zero-distance data sample skipped)."""
    P = _xyz(P)
    X0 = _xyz(X0)
    m = X0.shape[0]
    out = np.empty_like(X0)
    iso = np.empty(max(m, 1), dtype=np.uint32)
    fl = np.zeros(max(m, 1), dtype=np.uint8)
    prm = OrcParams(h, cutoff, mu, iterations, tol, eta, 1 if wlop else 0, 1 if store_f32 else 0)
    s = OrcSummary()
    rc = orc().orc_lop_project_flags(_ptr(P, _c_dbl_p), P.shape[0], _ptr(X0, _c_dbl_p), m,
                                     C.byref(prm), _ptr(out, _c_dbl_p), C.byref(s),
                                     _ptr(iso, _c_u32_p), _ptr(fl, _c_u8_p) if flags else None,
                                     threads)
    if rc:
        raise OracleError(rc)
    r = Result(out, s.iterations_run, bool(s.converged), s.isolated_events,
               s.coincident_pairs, iso[: s.n_isolated].copy(), s.interactions_attr,
               s.interactions_rep, s.last_max_disp)
    if flags:
        r.flags = fl[:m].copy()
    return r


def lop_sweep(P, X, h, cutoff=3.0, mu=0.4, eta=ETA_INV_CUBE, wlop=False, threads=0):
    """One Jacobi sweep: returns (X_next, isolated[u8], coincident[u32], max_disp)."""
    P = _xyz(P)
    X = _xyz(X)
    m = X.shape[0]
    nxt = np.empty_like(X)
    iso = np.zeros(max(m, 1), dtype=np.uint8)
    co = np.zeros(max(m, 1), dtype=np.uint32)
    md = C.c_double(0.0)
    prm = OrcParams(h, cutoff, mu, 1, 1e-7, eta, 1 if wlop else 0, 0)
    rc = orc().orc_lop_sweep(_ptr(P, _c_dbl_p), P.shape[0], _ptr(X, _c_dbl_p), m, C.byref(prm),
                             _ptr(nxt, _c_dbl_p), _ptr(iso, _c_u8_p), _ptr(co, _c_u32_p),
                             C.byref(md), threads)
    if rc:
        raise OracleError(rc)
    return nxt, iso[:m], co[:m], md.value


def lop_sweep_rows(P, X, rows, h, cutoff=3.0, mu=0.4, eta=ETA_INV_CUBE, wlop=False, threads=0):
    """One sweep from X for the query rows only (orc_lop_sweep_rows): returns
    (X_next[rows], counts[rows, 4]) with counts = (attraction interactions,
    repulsion interactions, coincident pairs, flags: 1 isolated, 2 anchored)."""
    P = _xyz(P)
    X = _xyz(X)
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    nr = rows.shape[0]
    nxt = np.empty((max(nr, 1), 3), dtype=np.float64)
    cnt = np.zeros((max(nr, 1), 4), dtype=np.int32)
    prm = OrcParams(h, cutoff, mu, 1, 1e-7, eta, 1 if wlop else 0, 0)
    rc = orc().orc_lop_sweep_rows(_ptr(P, _c_dbl_p), P.shape[0], _ptr(X, _c_dbl_p), X.shape[0],
                                  C.byref(prm), _ptr(rows, _c_u32_p), nr, _ptr(nxt, _c_dbl_p),
                                  cnt.ctypes.data_as(C.POINTER(C.c_int32)), threads)
    if rc:
        raise OracleError(rc)
    return nxt[:nr], cnt[:nr]


def radius_query_all(C_pts, Q, r, threads=0):
    """CSR (offsets[m+1], idx, dist) of SpatialIndex::radius_query for every query."""
    C_pts = _xyz(C_pts)
    Q = _xyz(Q)
    m = Q.shape[0]
    off = np.zeros(m + 1, dtype=np.uint64)
    lib = orc()
    rc = lib.orc_radius_query_all(_ptr(C_pts, _c_dbl_p), C_pts.shape[0], _ptr(Q, _c_dbl_p), m,
                                  r, _ptr(off, _c_u64_p), None, None, threads)
    if rc:
        raise OracleError(rc)
    tot = int(off[-1])
    idx = np.empty(max(tot, 1), dtype=np.uint32)
    dist = np.empty(max(tot, 1), dtype=np.float64)
    rc = lib.orc_radius_query_all(_ptr(C_pts, _c_dbl_p), C_pts.shape[0], _ptr(Q, _c_dbl_p), m,
                                  r, _ptr(off, _c_u64_p), _ptr(idx, _c_u32_p),
                                  _ptr(dist, _c_dbl_p), threads)
    if rc:
        raise OracleError(rc)
    return off, idx[:tot], dist[:tot]


def density_weights(C_pts, h, cutoff, threads=0):
    C_pts = _xyz(C_pts)
    v = np.empty(C_pts.shape[0], dtype=np.float64)
    rc = orc().orc_density_weights(_ptr(C_pts, _c_dbl_p), C_pts.shape[0], h, cutoff,
                                   _ptr(v, _c_dbl_p), threads)
    if rc:
        raise OracleError(rc)
    return v


def add_noise(xyz, sigma, seed):
    a = _xyz(xyz).copy()
    orc().orc_add_noise(_ptr(a, _c_dbl_p), a.shape[0], sigma, seed)
    return a


def plane(n, seed):
    a = np.empty((n, 3), dtype=np.float64)
    orc().orc_plane(_ptr(a, _c_dbl_p), n, seed)
    return a


def sphere(n, seed):
    a = np.empty((n, 3), dtype=np.float64)
    orc().orc_sphere(_ptr(a, _c_dbl_p), n, seed)
    return a


def generate_config(cfg: int, scale: float = 1.0):
    """(P, X0) of benchmark configuration cfg (orc_generate_config: the same draws
    as the product's pcs_generate_config, restated in the oracle so that the
    reference arm never loads the product library)."""
    n_p = np.zeros(1, dtype=np.uint64)
    n_x = np.zeros(1, dtype=np.uint64)
    lib = orc()
    if lib.orc_config_sizes(cfg, scale, _ptr(n_p, _c_u64_p), _ptr(n_x, _c_u64_p)):
        raise OracleError(1, f"config {cfg}")
    P = np.empty((int(n_p[0]), 3), dtype=np.float64)
    X0 = np.empty((int(n_x[0]), 3), dtype=np.float64)
    rc = lib.orc_generate_config(cfg, scale, _ptr(P, _c_dbl_p), _ptr(X0, _c_dbl_p))
    if rc:
        raise OracleError(rc)
    return P, X0


def theta(d, h, cutoff=3.0):
    return orc().orc_theta(d, h, cutoff)


# --- the unmodified reference (oracle/_ref) ------------------------------------

def ref_lop_project(P, X0, h, cutoff=3.0, mu=0.4, iterations=30, tol=1e-7,
                    eta=ETA_INV_CUBE) -> Result:
    """pcs::lop_project of the reference build (eta = ETA_NEG_LINEAR: the
    reference's lop.cpp with |eta'| = 1, see REF_ETAR_PATH)."""
    P = _xyz(P)
    X0 = _xyz(X0)
    m = X0.shape[0]
    out = np.empty_like(X0)
    iso = np.empty(max(m, 1), dtype=np.uint32)
    s = RefSummary()
    lib = ref(eta)
    rc = lib.ref_lop_project(_ptr(P, _c_dbl_p), P.shape[0], _ptr(X0, _c_dbl_p), m, h, cutoff,
                             mu, iterations, tol, _ptr(out, _c_dbl_p), C.byref(s),
                             _ptr(iso, _c_u32_p))
    if rc:
        raise OracleError(rc, lib.ref_last_error().decode())
    return Result(out, s.iterations_run, bool(s.converged), s.isolated_events,
                  s.coincident_pairs, iso[: s.n_isolated].copy())


def ref_radius_query_all(C_pts, Q, r):
    C_pts = _xyz(C_pts)
    Q = _xyz(Q)
    m = Q.shape[0]
    off = np.zeros(m + 1, dtype=np.uint64)
    lib = ref()
    rc = lib.ref_radius_query_all(_ptr(C_pts, _c_dbl_p), C_pts.shape[0], _ptr(Q, _c_dbl_p), m,
                                  r, _ptr(off, _c_u64_p), None, None)
    if rc:
        raise OracleError(rc, lib.ref_last_error().decode())
    tot = int(off[-1])
    idx = np.empty(max(tot, 1), dtype=np.uint32)
    dist = np.empty(max(tot, 1), dtype=np.float64)
    rc = lib.ref_radius_query_all(_ptr(C_pts, _c_dbl_p), C_pts.shape[0], _ptr(Q, _c_dbl_p), m,
                                  r, _ptr(off, _c_u64_p), _ptr(idx, _c_u32_p),
                                  _ptr(dist, _c_dbl_p))
    if rc:
        raise OracleError(rc, lib.ref_last_error().decode())
    return off, idx[:tot], dist[:tot]


def ref_generate_surface(kind: int, n: int, seed: int) -> np.ndarray:
    a = np.empty((n, 3), dtype=np.float64)
    rc = ref().ref_generate_surface(kind, n, seed, _ptr(a, _c_dbl_p))
    if rc:
        raise OracleError(rc)
    return a


def ref_add_noise(xyz, sigma, seed):
    a = _xyz(xyz).copy()
    rc = ref().ref_add_noise(_ptr(a, _c_dbl_p), a.shape[0], sigma, seed)
    if rc:
        raise OracleError(rc)
    return a


def ref_index_build_ms(P) -> float:
    P = _xyz(P)
    return float(ref().ref_index_build_ms(_ptr(P, _c_dbl_p), P.shape[0]))


# --- deviation metrics (proj/src/spatial.cpp:119-158, proj/src/metrics.cpp) -------
def _dptr(a):
    return a.ctypes.data_as(_c_dbl_p) if a.size else None


def nearest_all(C_pts, Q, threads=0):
    """Restated SpatialIndex::nearest for every query: (idx uint32, dist)."""
    Cc, Qq = _xyz(C_pts), _xyz(Q)
    m = Qq.shape[0]
    idx = np.zeros(max(m, 1), np.uint32)
    dist = np.zeros(max(m, 1), np.float64)
    st = orc().orc_nearest_all(_dptr(Cc), Cc.shape[0], _dptr(Qq), m, _ptr(idx, _c_u32_p),
                               _ptr(dist, _c_dbl_p), threads)
    if st:
        raise OracleError(st, "nearest")
    return idx[:m], dist[:m]


def deviation(cloud, reference, threads=0):
    """Restated pcs::deviation: ({n, mean, rms, max} array, distances)."""
    Cc, Rr = _xyz(cloud), _xyz(reference)
    out = np.zeros(4, np.float64)
    dist = np.zeros(max(Cc.shape[0], 1), np.float64)
    st = orc().orc_deviation(_dptr(Cc), Cc.shape[0], _dptr(Rr), Rr.shape[0], _ptr(out, _c_dbl_p),
                             _ptr(dist, _c_dbl_p), threads)
    if st:
        raise OracleError(st, "deviation")
    return out, dist[: Cc.shape[0]]


def point_triangle_distance(p, tri) -> float:
    pp = np.ascontiguousarray(np.asarray(p, np.float64).reshape(3))
    tt = np.ascontiguousarray(np.asarray(tri, np.float64).reshape(9))
    return orc().orc_point_triangle_distance(_ptr(pp, _c_dbl_p), _ptr(tt, _c_dbl_p))


def deviation_to_mesh(cloud, triangles, threads=0):
    Cc = _xyz(cloud)
    T = np.ascontiguousarray(np.asarray(triangles, np.float64).reshape(-1, 9))
    out = np.zeros(4, np.float64)
    dist = np.zeros(max(Cc.shape[0], 1), np.float64)
    st = orc().orc_deviation_to_mesh(_dptr(Cc), Cc.shape[0], _dptr(T), T.shape[0],
                                     _ptr(out, _c_dbl_p), _ptr(dist, _c_dbl_p), threads)
    if st:
        raise OracleError(st, "deviation_to_mesh")
    return out, dist[: Cc.shape[0]]


def ref_nearest_all(C_pts, Q, threads=0):
    Cc, Qq = _xyz(C_pts), _xyz(Q)
    m = Qq.shape[0]
    idx = np.zeros(max(m, 1), np.uint32)
    dist = np.zeros(max(m, 1), np.float64)
    st = ref().ref_nearest_all(_dptr(Cc), Cc.shape[0], _dptr(Qq), m, _ptr(idx, _c_u32_p),
                               _ptr(dist, _c_dbl_p), threads)
    if st:
        raise OracleError(st, ref().ref_last_error().decode())
    return idx[:m], dist[:m]


def ref_deviation(cloud, reference):
    Cc, Rr = _xyz(cloud), _xyz(reference)
    out = np.zeros(4, np.float64)
    dist = np.zeros(max(Cc.shape[0], 1), np.float64)
    st = ref().ref_deviation(_dptr(Cc), Cc.shape[0], _dptr(Rr), Rr.shape[0], _ptr(out, _c_dbl_p),
                             _ptr(dist, _c_dbl_p))
    if st:
        raise OracleError(st, ref().ref_last_error().decode())
    return out, dist[: Cc.shape[0]]


def ref_deviation_to_mesh(cloud, triangles):
    Cc = _xyz(cloud)
    T = np.ascontiguousarray(np.asarray(triangles, np.float64).reshape(-1, 9))
    out = np.zeros(4, np.float64)
    dist = np.zeros(max(Cc.shape[0], 1), np.float64)
    st = ref().ref_deviation_to_mesh(_dptr(Cc), Cc.shape[0], _dptr(T), T.shape[0],
                                     _ptr(out, _c_dbl_p), _ptr(dist, _c_dbl_p))
    if st:
        raise OracleError(st, ref().ref_last_error().decode())
    return out, dist[: Cc.shape[0]]


def ref_point_triangle_distance(p, tri) -> float:
    pp = np.ascontiguousarray(np.asarray(p, np.float64).reshape(3))
    tt = np.ascontiguousarray(np.asarray(tri, np.float64).reshape(9))
    return ref().ref_point_triangle_distance(_ptr(pp, _c_dbl_p), _ptr(tt, _c_dbl_p))


# --- cloud IO through the reference (proj/src/io.cpp) ------------------------------
def ref_format_cloud(xyz, fmt=0) -> bytes:
    X = _xyz(xyz)
    n = C.c_uint64(0)
    ref().ref_format_cloud(_dptr(X), X.shape[0], fmt, None, 0, C.byref(n))
    buf = C.create_string_buffer(max(n.value, 1))
    st = ref().ref_format_cloud(_dptr(X), X.shape[0], fmt, buf, n.value, C.byref(n))
    if st:
        raise OracleError(st, ref().ref_last_error().decode())
    return buf.raw[: n.value]


def ref_parse_cloud(text: bytes, fmt=0):
    """(points, None) or (None, (line, message)) for a ParseError."""
    cap = len(text) // 6 + 1
    out = np.zeros((cap, 3), np.float64)
    n = C.c_uint64(0)
    line = C.c_int64(0)
    st = ref().ref_parse_cloud(text, len(text), fmt, _ptr(out, _c_dbl_p), cap, C.byref(n),
                               C.byref(line))
    if st == 10:
        return None, (line.value, ref().ref_last_error().decode())
    if st:
        raise OracleError(st, ref().ref_last_error().decode())
    return out[: n.value], None
