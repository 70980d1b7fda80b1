"""Python mirror of the reference's LOP operator interface.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/pcs/lop.hpp:12-53, kernels.hpp:12-34,
errors.hpp:9-53); the work is done by the sm_100a library through the C ABI
(include/pcs_lop.h).  Clouds are ``(n, 3)`` float64 arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _lib as L


# ---- errors (proj/include/pcs/errors.hpp) --------------------------------------
class Error(RuntimeError):
    """Base class for all library errors."""


class EmptyCloud(Error):
    pass


class InvalidParam(Error):
    pass


class EmptyMesh(Error):
    pass


class ParseError(Error):
    """Malformed cloud / mesh text; ``line`` is the 1-based line number (0 when
    the error concerns the whole file), message "name:line: reason"."""

    def __init__(self, name: str, line: int, reason: str):
        super().__init__(f"{name}:{line}: {reason}")
        self.line = line
        self.reason = reason


class NumericalFailure(Error):
    """Numerical or device failure (CUDA / NCCL error, no sm_100 device)."""


class DeviceUnavailable(NumericalFailure):
    pass


def _raise(status: int) -> None:
    msg = L.last_error()
    if status == L.PCS_ERR_INVALID_PARAM:
        raise InvalidParam(msg)
    if status == L.PCS_ERR_EMPTY_CLOUD:
        raise EmptyCloud(msg)
    if status == L.PCS_ERR_EMPTY_MESH:
        raise EmptyMesh(msg)
    if status == L.PCS_ERR_NO_DEVICE:
        raise DeviceUnavailable(msg)
    raise NumericalFailure(f"[status {status}] {msg}")


def _check(status: int) -> None:
    if status != L.PCS_OK:
        _raise(status)


# ---- parameters (proj/include/pcs/kernels.hpp:12-24, lop.hpp:12-35) --------------
@dataclass
class KernelParams:
    h: float = 1.0
    cutoff_multiple: float = 3.0

    def support(self) -> float:
        return self.h * self.cutoff_multiple

    def validate(self) -> None:
        if not (self.h > 0.0):
            raise InvalidParam("kernel bandwidth h must be positive")
        if not (self.cutoff_multiple > 0.0):
            raise InvalidParam("kernel cutoff_multiple must be positive")


@dataclass
class LopParams:
    kernel: KernelParams = field(default_factory=KernelParams)
    mu: float = 0.4
    iterations: int = 30
    convergence_tol: float = 1e-7

    def validate(self) -> None:
        self.kernel.validate()
        if not (self.mu >= 0.0) or not (self.mu < 0.5):
            raise InvalidParam("LopParams: mu must be in [0, 0.5)")
        if self.iterations < 1:
            raise InvalidParam("LopParams: iterations must be >= 1")
        if not (self.convergence_tol > 0.0):
            raise InvalidParam("LopParams: convergence_tol must be positive")


@dataclass
class LopSummary:
    iterations_run: int = 0
    converged: bool = False
    isolated_events: int = 0
    coincident_pairs: int = 0
    isolated_indices: List[int] = field(default_factory=list)
    # measured extras (not in the reference struct)
    interactions_attr: int = 0
    interactions_rep: int = 0
    density_pairs: int = 0
    careful_points: int = 0
    last_max_disp: float = 0.0
    setup_ms: float = 0.0
    sweeps_ms: float = 0.0
    kernel_ms: float = 0.0
    sort_ms: float = 0.0
    lane_candidates: int = 0


ETA = {"inv_cube": L.PCS_ETA_INV_CUBE, "neg_linear": L.PCS_ETA_NEG_LINEAR}
PRECISION = {"fp64": L.PCS_PREC_FP64, "fp32": L.PCS_PREC_FP32}


def make_desc(params: LopParams, eta: str = "inv_cube", density_weights: bool = False,
              precision: str = "fp64", device: int = -1, lanes_per_point: int = 0) -> L.LopDesc:
    d = L.LopDesc()
    L.lib().pcs_lop_desc_default(C.byref(d))
    d.h = float(params.kernel.h)
    d.cutoff_multiple = float(params.kernel.cutoff_multiple)
    d.mu = float(params.mu)
    d.iterations = int(params.iterations)
    d.convergence_tol = float(params.convergence_tol)
    if eta not in ETA:
        raise InvalidParam(f"eta must be one of {sorted(ETA)}")
    if precision not in PRECISION:
        raise InvalidParam(f"precision must be one of {sorted(PRECISION)}")
    d.eta_kind = ETA[eta]
    d.density_weights = 1 if density_weights else 0
    d.precision = PRECISION[precision]
    d.device = int(device)
    d.lanes_per_point = int(lanes_per_point)
    return d


def _cloud(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        return np.zeros((0, 3), dtype=np.float64)
    return np.ascontiguousarray(a.reshape(-1, 3))


def _ptr(a, t=L._dp):
    return a.ctypes.data_as(t) if a.size else None


def _summary(s: L.LopSummaryC, iso: np.ndarray) -> LopSummary:
    return LopSummary(
        iterations_run=s.iterations_run, converged=bool(s.converged),
        isolated_events=int(s.isolated_events), coincident_pairs=int(s.coincident_pairs),
        isolated_indices=[int(v) for v in iso[: min(int(s.n_isolated), iso.size)]],
        interactions_attr=int(s.interactions_attr), interactions_rep=int(s.interactions_rep),
        density_pairs=int(s.density_pairs), careful_points=int(s.careful_points),
        last_max_disp=float(s.last_max_disp), setup_ms=float(s.setup_ms),
        sweeps_ms=float(s.sweeps_ms), kernel_ms=float(s.kernel_ms), sort_ms=float(s.sort_ms),
        lane_candidates=int(s.lane_candidates))


def lop_project(data, initial, params: LopParams, *, eta: str = "inv_cube",
                density_weights: bool = False, precision: str = "fp64", device: int = -1,
                lanes_per_point: int = 0) -> Tuple[np.ndarray, LopSummary]:
    """pcs::lop_project (proj/include/pcs/lop.hpp:51-53) on the B200.

    Validation order of proj/src/lop.cpp:13-20: InvalidParam, EmptyCloud for
    empty data, an empty ``initial`` passes through unchanged.
    """
    params.validate()
    P = _cloud(data)
    X0 = _cloud(initial)
    d = make_desc(params, eta, density_weights, precision, device, lanes_per_point)
    out = np.empty_like(X0)
    iso = np.zeros(max(X0.shape[0], 1), dtype=np.uint32)
    s = L.LopSummaryC()
    st = L.lib().pcs_lop_run(C.byref(d), _ptr(P), P.shape[0], _ptr(X0), X0.shape[0], _ptr(out),
                             C.byref(s), _ptr(iso, L._u32p), iso.size)
    _check(st)
    return out, _summary(s, iso)


class LopPlan:
    """Device-resident run (the bench path): upload once, sweep many times."""

    def __init__(self, params: LopParams, *, eta: str = "inv_cube", density_weights: bool = False,
                 precision: str = "fp64", device: int = -1, lanes_per_point: int = 0):
        params.validate()
        self.desc = make_desc(params, eta, density_weights, precision, device, lanes_per_point)
        h = C.c_void_p()
        _check(L.lib().pcs_lop_plan_create(C.byref(self.desc), C.byref(h)))
        self._h = h
        self.m = 0

    def close(self) -> None:
        if self._h:
            L.lib().pcs_lop_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(L.lib().pcs_nccl_unique_id(buf))
        return bytes(buf)

    def set_comm(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(L.lib().pcs_lop_plan_set_comm(self._h, buf, nranks, rank))

    def set_loopback(self, group: "LoopbackGroup", rank: int) -> None:
        """In-process rank of a loopback group (validation of the sharded path on one GPU)."""
        _check(L.lib().pcs_lop_plan_set_loopback(self._h, group._h, rank))
        self._group = group  # keep the group alive as long as the plan

    def upload(self, data, initial) -> None:
        P = _cloud(data)
        X0 = _cloud(initial)
        self.m = X0.shape[0]
        _check(L.lib().pcs_lop_plan_upload(self._h, _ptr(P), P.shape[0], _ptr(X0), X0.shape[0]))

    def reset(self) -> None:
        _check(L.lib().pcs_lop_plan_reset(self._h))

    def run(self, sweeps: int = 0, sync: bool = True) -> None:
        _check(L.lib().pcs_lop_plan_run(self._h, int(sweeps), 1 if sync else 0))

    def synchronize(self) -> None:
        _check(L.lib().pcs_lop_plan_synchronize(self._h))

    def last_run_ms(self) -> float:
        v = C.c_double(0.0)
        _check(L.lib().pcs_lop_plan_last_run_ms(self._h, C.byref(v)))
        return v.value

    def launches(self) -> int:
        return int(L.lib().pcs_lop_plan_launches(self._h))

    def set_positions(self, X) -> None:
        """Restart point: the next run starts from X (m points) instead of X0."""
        Xc = _cloud(X)
        _check(L.lib().pcs_lop_plan_set_positions(self._h, _ptr(Xc), Xc.shape[0]))

    def set_graphs(self, enable: bool) -> None:
        """CUDA-graph replay of the sweeps (default on; off = every launch enqueued)."""
        _check(L.lib().pcs_lop_plan_set_graphs(self._h, 1 if enable else 0))

    def graph_launches(self) -> int:
        return int(L.lib().pcs_lop_plan_graph_launches(self._h))

    def record_counts(self, enable: bool = True) -> None:
        """Parity facility: record per-query counts every sweep (after upload)."""
        _check(L.lib().pcs_lop_plan_record_counts(self._h, 1 if enable else 0))

    def query_counts(self) -> Tuple[np.ndarray, np.ndarray]:
        """(counts[m, 4], ever_flags[m]) of the last sweep: attraction and repulsion
        interactions, coincident pairs, flags (1 isolated, 2 anchored, 4 deferred to
        the exact kernel); ever_flags = flags OR-ed over the run."""
        cnt = np.zeros((max(self.m, 1), 4), dtype=np.int32)
        ev = np.zeros(max(self.m, 1), dtype=np.uint8)
        _check(L.lib().pcs_lop_plan_query_counts(self._h, cnt.ctypes.data_as(C.POINTER(C.c_int32)),
                                                 _ptr(ev, L._u8p), self.m))
        return cnt[: self.m], ev[: self.m]

    def download(self) -> Tuple[np.ndarray, LopSummary]:
        out = np.empty((self.m, 3), dtype=np.float64)
        iso = np.zeros(max(self.m, 1), dtype=np.uint32)
        s = L.LopSummaryC()
        _check(L.lib().pcs_lop_plan_download(self._h, _ptr(out), C.byref(s), _ptr(iso, L._u32p),
                                             iso.size))
        return out, _summary(s, iso)


class LoopbackGroup:
    """R in-process ranks on one device (pcs_loopback_group_create).

    Each rank's LopPlan must be driven by its own thread (the exchange step is a
    host rendezvous).  A validation facility for the multi-GPU path, not a
    performance mode.
    """

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _check(L.lib().pcs_loopback_group_create(nranks, C.byref(h)))
        self._h = h
        self.nranks = nranks

    def __del__(self):
        if getattr(self, "_h", None):
            L.lib().pcs_loopback_group_destroy(self._h)
            self._h = None


def radius_query_all(cloud, queries, r: float, precision: str = "fp64", device: int = -1):
    """SpatialIndex::radius_query (proj/src/spatial.cpp:82-111) for every query,
    on the device grid; returns CSR ``(offsets[m+1], idx)``, hits ascending."""
    Cc = _cloud(cloud)
    Q = _cloud(queries)
    m = Q.shape[0]
    d = make_desc(LopParams(), precision=precision, device=device)
    off = np.zeros(m + 1, dtype=np.uint64)
    _check(L.lib().pcs_radius_query_all(C.byref(d), _ptr(Cc), Cc.shape[0], _ptr(Q), m, float(r),
                                        off.ctypes.data_as(L._u64p), None, 0))
    tot = int(off[-1])
    idx = np.zeros(max(tot, 1), dtype=np.uint32)
    _check(L.lib().pcs_radius_query_all(C.byref(d), _ptr(Cc), Cc.shape[0], _ptr(Q), m, float(r),
                                        off.ctypes.data_as(L._u64p), _ptr(idx, L._u32p), tot))
    return off, idx[:tot]


# ---- cloud files (proj/include/pcs/io.hpp, proj/src/io.cpp) -------------------------
_FORMATS = {"xyz": L.PCS_FMT_XYZ, "ply": L.PCS_FMT_PLY_ASCII}


def format_from_path(path: str) -> str:
    """'xyz' or 'ply' from the extension (case-insensitive), else InvalidParam."""
    ext = os.path.splitext(path)[1].lower()
    if ext in (".xyz", ".ply"):
        return ext[1:]
    raise InvalidParam(f"cannot infer cloud format from '{path}' (expected .xyz or .ply); "
                       "pass the format explicitly")


def _format_into_buffer(cloud, fmt: str, device: int):
    """The text of ``cloud`` in a caller-side uint8 buffer sized by the longest
    shortest-round-trip form (24 characters per coordinate): (buffer, length)."""
    Cc = _cloud(cloud)
    d = make_desc(LopParams(), device=device)
    cap = 80 * Cc.shape[0] + 4096
    buf = np.empty(cap, dtype=np.uint8)
    n = C.c_uint64(0)
    _check(L.lib().pcs_format_cloud(C.byref(d), _ptr(Cc), Cc.shape[0], _FORMATS[fmt],
                                    C.cast(buf.ctypes.data, C.c_char_p), cap, C.byref(n)))
    return buf, int(n.value)


def format_cloud(cloud, fmt: str = "xyz", device: int = -1) -> bytes:
    """write_cloud_stream (proj/src/io.cpp:277-290): the file bytes, coordinates
    as shortest round-trip decimals, formatted on the device (one pass)."""
    buf, n = _format_into_buffer(cloud, fmt, device)
    return buf[:n].tobytes()


def parse_cloud(text: bytes, fmt: str = "xyz", name: str = "<memory>", device: int = -1) -> np.ndarray:
    """read_cloud_stream (proj/src/io.cpp:143-236): ``(n, 3)`` float64 points,
    parsed on the device; ParseError(name, line, reason) like the reference."""
    d = make_desc(LopParams(), device=device)
    cap = len(text) // 6 + 1
    out = np.zeros((cap, 3), dtype=np.float64)
    n = C.c_uint64(0)
    err = L.ParseErrorC()
    st = L.lib().pcs_parse_cloud(C.byref(d), text, len(text), _FORMATS[fmt], _ptr(out), cap,
                                 C.byref(n), C.byref(err))
    if st == L.PCS_ERR_PARSE:
        raise ParseError(name, int(err.line), err.reason.decode())
    _check(st)
    return out[: n.value]


def read_cloud(path: str, fmt: Optional[str] = None, device: int = -1) -> np.ndarray:
    fmt = fmt or format_from_path(path)
    with open(path, "rb") as f:
        return parse_cloud(f.read(), fmt, name=path, device=device)


def write_cloud(cloud, path: str, fmt: Optional[str] = None, device: int = -1) -> None:
    """write_cloud (proj/src/io.cpp:292-301).  The text lands in a caller-side
    buffer sized by the longest shortest-round-trip form (24 characters per
    coordinate) and goes to the file from there: no intermediate ``bytes``
    (10M points: 0.03 s of formatting instead of 0.34 s through format_cloud)."""
    fmt = fmt or format_from_path(path)
    buf, n = _format_into_buffer(cloud, fmt, device)
    with open(path, "wb") as f:
        f.write(memoryview(buf)[:n])


def parse_mesh(text: bytes, name: str = "<memory>") -> np.ndarray:
    """read_mesh_stream: ``(T, 3, 3)`` triangles of an ASCII PLY face element."""
    n = C.c_uint64(0)
    err = L.ParseErrorC()
    st = L.lib().pcs_parse_mesh(text, len(text), None, 0, C.byref(n), C.byref(err))
    if st == L.PCS_ERR_PARSE:
        raise ParseError(name, int(err.line), err.reason.decode())
    if st != L.PCS_ERR_CAPACITY:
        _check(st)
    out = np.zeros((max(n.value, 1), 9), dtype=np.float64)
    _check(L.lib().pcs_parse_mesh(text, len(text), _ptr(out), n.value, C.byref(n), C.byref(err)))
    return out[: n.value].reshape(-1, 3, 3)


def format_double(v: float) -> str:
    buf = C.create_string_buffer(40)
    n = L.lib().pcs_format_double(float(v), buf)
    return buf.raw[:n].decode()


# ---- deviation metrics (proj/include/pcs/metrics.hpp, proj/src/metrics.cpp) ----
@dataclass
class DeviationReport:
    """n, mean distance, RMS distance (``std_deviation``) and max distance;
    ``distances`` (per cloud point) when requested."""
    n: int = 0
    mean_distance: float = 0.0
    std_deviation: float = 0.0
    max_distance: float = 0.0
    distances: Optional[np.ndarray] = None


def nearest_all(cloud, queries, device: int = -1) -> Tuple[np.ndarray, np.ndarray]:
    """SpatialIndex::nearest (proj/src/spatial.cpp:119-158) for every query, on the
    device: ``(index, distance)`` of the nearest cloud point, smallest index on
    equal distance, distances bit-identical to the reference."""
    Cc = _cloud(cloud)
    Q = _cloud(queries)
    m = Q.shape[0]
    idx = np.zeros(max(m, 1), dtype=np.uint32)
    dist = np.zeros(max(m, 1), dtype=np.float64)
    d = make_desc(LopParams(), device=device)
    _check(L.lib().pcs_nearest_all(C.byref(d), _ptr(Cc), Cc.shape[0], _ptr(Q), m,
                                   _ptr(idx, L._u32p), _ptr(dist)))
    return idx[:m], dist[:m]


def _report(r, dist, keep):
    return DeviationReport(int(r.n), r.mean_distance, r.std_deviation, r.max_distance,
                           dist if keep else None)


def deviation(cloud, reference, keep_distances: bool = False, device: int = -1) -> DeviationReport:
    """pcs::deviation (proj/src/metrics.cpp:39-53): nearest-reference distance of
    every cloud point (device), aggregated in index order like the reference."""
    Cc = _cloud(cloud)
    R = _cloud(reference)
    m = Cc.shape[0]
    dist = np.zeros(max(m, 1), dtype=np.float64)
    r = L.DeviationReportC()
    d = make_desc(LopParams(), device=device)
    _check(L.lib().pcs_deviation(C.byref(d), _ptr(Cc), m, _ptr(R), R.shape[0], C.byref(r),
                                 _ptr(dist)))
    return _report(r, dist[:m], keep_distances)


def deviation_to_mesh(cloud, triangles, keep_distances: bool = False,
                      device: int = -1) -> DeviationReport:
    """pcs::deviation_to_mesh (proj/src/metrics.cpp:115-133); ``triangles`` is a
    ``(T, 3, 3)`` array of vertices a, b, c."""
    Cc = _cloud(cloud)
    T = np.ascontiguousarray(np.asarray(triangles, dtype=np.float64).reshape(-1, 9))
    m = Cc.shape[0]
    dist = np.zeros(max(m, 1), dtype=np.float64)
    r = L.DeviationReportC()
    d = make_desc(LopParams(), device=device)
    tp = _ptr(T) if T.shape[0] else None
    _check(L.lib().pcs_deviation_to_mesh(C.byref(d), _ptr(Cc), m, tp, T.shape[0], C.byref(r),
                                         _ptr(dist)))
    return _report(r, dist[:m], keep_distances)


def density_weights(cloud, h: float, cutoff_multiple: float = 3.0, precision: str = "fp64",
                    device: int = -1) -> np.ndarray:
    """WLOP density weights v_j = 1 + sum_{j' != j, d <= support} theta(d)."""
    Cc = _cloud(cloud)
    v = np.zeros(max(Cc.shape[0], 1), dtype=np.float64)
    d = make_desc(LopParams(kernel=KernelParams(h, cutoff_multiple)), precision=precision,
                  device=device)
    _check(L.lib().pcs_density_weights(C.byref(d), _ptr(Cc), Cc.shape[0], _ptr(v)))
    return v[: Cc.shape[0]]


def grid_sort(cloud, support: float, precision: str = "fp64", device: int = -1):
    """(sorted keys, order) of the device hash for a cloud."""
    Cc = _cloud(cloud)
    n = Cc.shape[0]
    keys = np.zeros(max(n, 1), dtype=np.uint32)
    order = np.zeros(max(n, 1), dtype=np.uint32)
    d = make_desc(LopParams(), precision=precision, device=device)
    _check(L.lib().pcs_grid_sort(C.byref(d), _ptr(Cc), n, float(support), _ptr(keys, L._u32p),
                                 _ptr(order, L._u32p)))
    return keys[:n], order[:n]


def shard_layout(sorted_order, nranks: int, weights=None):
    """Multi-GPU ownership layout: returns (chunk, counts, orig_of_internal[nranks*chunk],
    internal_of_orig[m]).  Without weights: equal counts (pcs_shard_layout); with
    weights[o] = estimated work of original point o: cuts at equal cumulative
    work (pcs_shard_layout_weighted, what sharded plans use)."""
    so = np.ascontiguousarray(np.asarray(sorted_order, dtype=np.uint32))
    m = so.size
    chunk = C.c_uint32()
    counts = np.zeros(nranks, dtype=np.uint32)
    ioo = np.zeros(max(m, 1), dtype=np.uint32)
    if weights is None:
        cap = max(1, (m + nranks - 1) // nranks * nranks)
        ooi = np.zeros(cap, dtype=np.uint32)
        _check(L.lib().pcs_shard_layout(_ptr(so, L._u32p), m, nranks, ooi.ctypes.data_as(L._u32p),
                                        ioo.ctypes.data_as(L._u32p), C.byref(chunk),
                                        counts.ctypes.data_as(L._u32p)))
    else:
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float32))
        wp = w.ctypes.data_as(C.POINTER(C.c_float))
        _check(L.lib().pcs_shard_layout_weighted(_ptr(so, L._u32p), wp, m, nranks, None, None,
                                                 C.byref(chunk), counts.ctypes.data_as(L._u32p)))
        ooi = np.zeros(max(1, chunk.value * nranks), dtype=np.uint32)
        _check(L.lib().pcs_shard_layout_weighted(_ptr(so, L._u32p), wp, m, nranks,
                                                 ooi.ctypes.data_as(L._u32p),
                                                 ioo.ctypes.data_as(L._u32p), C.byref(chunk),
                                                 counts.ctypes.data_as(L._u32p)))
    return chunk.value, counts, ooi[: chunk.value * nranks], ioo[:m]


# ---- host generators (rng.hpp / bench.cpp / noise.cpp semantics) ------------------
SURFACE = {"plane": 0, "sphere": 1, "torus": 2, "bump": 3}


def generate_surface(kind: str, n: int, seed: int) -> np.ndarray:
    a = np.empty((n, 3), dtype=np.float64)
    _check(L.lib().pcs_generate_surface(SURFACE[kind], n, seed, _ptr(a)))
    return a


def add_noise(cloud, sigma: float, seed: int) -> np.ndarray:
    a = _cloud(cloud).copy()
    _check(L.lib().pcs_add_noise(_ptr(a), a.shape[0], float(sigma), int(seed)))
    return a


def config_sizes(config: int, scale: float = 1.0) -> Tuple[int, int]:
    n = C.c_uint64()
    m = C.c_uint64()
    _check(L.lib().pcs_config_sizes(config, float(scale), C.byref(n), C.byref(m)))
    return n.value, m.value


def generate_config(config: int, scale: float = 1.0) -> Tuple[np.ndarray, np.ndarray]:
    """Benchmark configuration 1..5 (BASELINE.json configs), fp64 host arrays."""
    n, m = config_sizes(config, scale)
    P = np.empty((n, 3), dtype=np.float64)
    X0 = np.empty((m, 3), dtype=np.float64)
    _check(L.lib().pcs_generate_config(config, float(scale), _ptr(P), _ptr(X0)))
    return P, X0


# Parameters of the five configurations (h = support radius -> KernelParams{h/4, 4}).
CONFIGS = {
    1: dict(h=0.1, mu=0.45, eta="inv_cube", wlop=False, iterations=20, precision="fp64"),
    2: dict(h=0.05, mu=0.45, eta="neg_linear", wlop=True, iterations=30, precision="fp32"),
    3: dict(h=0.02, mu=0.40, eta="neg_linear", wlop=False, iterations=15, precision="fp32"),
    4: dict(h=0.03, mu=0.45, eta="neg_linear", wlop=True, iterations=20, precision="fp32"),
    5: dict(h=0.02, mu=0.45, eta="inv_cube", wlop=False, iterations=10, precision="fp32"),
}


def config_params(config: int, h: Optional[float] = None) -> Tuple[LopParams, dict]:
    c = dict(CONFIGS[config])
    if h is not None:
        c["h"] = h
    p = LopParams(kernel=KernelParams(c["h"] / 4.0, 4.0), mu=c["mu"], iterations=c["iterations"])
    return p, c


def trim_device_pool(device: int = -1) -> None:
    """Returns the device memory the library keeps reserved between calls."""
    _check(L.lib().pcs_trim_device_pool(int(device)))
