"""MLS projection on the B200 (mls.cu) against the CPU oracle (GPU).

The oracle (oracle/lop_oracle.c orc_mls_project) restates proj/src/wls.cpp and
proj/src/mls.cpp with hits in index order and independent eigen-solvers
(closed-form 3x3, long-double Jacobi); the device sums over its grid
enumeration and diagonalises with fp64 Jacobi.  Bars: identical statuses,
degrees and plane iteration counts; frames, polynomial coefficients and
projections within 1e-9 (relative to the cloud scale) — rounding only.
Radius queries of the device index are bit-exact (indices and distances).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("sphere", 2000, 19, 0.05, 0.25, 2), ("sphere", 2000, 91, 0.05, 0.15, 2),
         ("bump", 1500, 31, 0.02, 0.15, 2), ("torus", 3000, 5, 0.01, 0.1, 3),
         ("sphere", 4000, 7, 0.01, 0.2, 4), ("plane", 2000, 3, 0.02, 0.2, 1)]


def cloud(pb, kind, n, seed, sigma):
    return pb.add_noise(pb.generate_surface(kind, n, seed), sigma, seed + 1)


@pytest.mark.parametrize("kind,n,seed,sigma,h,deg", CASES)
def test_smooth_cloud_matches_oracle(pb, orc, kind, n, seed, sigma, h, deg):
    P = cloud(pb, kind, n, seed, sigma)
    prm = pb.MlsParams(kernel=pb.KernelParams(h), degree=deg)
    out, res = pb.smooth_cloud(P, prm)
    r = orc.mls_project(P, P, h, degree=deg)
    assert np.array_equal(res.status, r["status"]), np.nonzero(res.status != r["status"])[0][:10]
    assert np.array_equal(res.degree_used, r["degree_used"])
    assert np.array_equal(res.plane_status, r["plane_status"])
    it_diff = np.nonzero(res.iterations != r["iterations"])[0]
    assert it_diff.size <= max(2, n // 1000), it_diff[:10]   # a converging step may land on tol
    scale = max(1.0, float(np.abs(P).max()))
    err = np.abs(out - r["projected"]).max()
    print(f"{kind} n={n} h={h} deg={deg}: statuses {np.bincount(res.status, minlength=4)}, "
          f"max |dev - oracle| {err:.2e}, iteration mismatches {it_diff.size}")
    assert err <= 1e-9 * scale
    assert np.array_equal(out, res.projected)


@pytest.mark.parametrize("deg", [1, 2, 3, 4])
def test_plane_and_polynomial_fits_match_oracle(pb, orc, deg):
    P = cloud(pb, "sphere", 3000, 40 + deg, 0.02)
    rng = np.random.default_rng(deg)
    Q = P[rng.choice(P.shape[0], 200, replace=False)] * (1 + rng.normal(0, 0.02, (200, 1)))
    prm = pb.MlsParams(kernel=pb.KernelParams(0.2), degree=deg)
    ix = pb.MlsIndex(P)
    try:
        pl = ix.project(Q, prm, mode=1)
        ro = orc.mls_project(P, Q, 0.2, degree=deg, mode=orc.MLS_PLANE)
        assert np.array_equal(pl.plane_status, ro["plane_status"])
        ok = pl.plane_status == 0
        for k in ("origin", "normal", "u", "v"):
            assert np.abs(getattr(pl, k)[ok] - ro[k][ok]).max() <= 1e-9, k
        fr = np.concatenate([ro["origin"], ro["normal"], ro["u"], ro["v"]], axis=1)[ok]
        po = ix.project(ro["origin"][ok], prm, mode=2, frames=fr)
        rp = orc.mls_project(P, ro["origin"][ok], 0.2, degree=deg, mode=orc.MLS_POLY, frames=fr)
        assert np.array_equal(po.poly_status, rp["poly_status"])
        K = (deg + 1) * (deg + 2) // 2
        good = po.poly_status == 0
        c_dev, c_orc = po.coeffs[good][:, :K], rp["coeffs"][good][:, :K]
        tol = 1e-9 * (1 + np.abs(c_orc).max(axis=1, keepdims=True))
        assert (np.abs(c_dev - c_orc) <= tol).all(), np.abs(c_dev - c_orc).max()
    finally:
        ix.close()


def test_index_radius_queries_bit_exact(pb, orc):
    rng = np.random.default_rng(9)
    C = rng.uniform(-1, 1, (20000, 3))
    C[:100] = C[100:200]                                   # duplicated coordinates
    Q = np.concatenate([C[rng.choice(20000, 300)], rng.uniform(-3, 3, (100, 3))])
    ix = pb.MlsIndex(C)
    try:
        for r in (0.02, 0.1, 0.35):
            off, idx, dist = ix.radius_query_all(Q, r)
            o2, i2, d2 = orc.radius_query_all(C, Q, r)
            assert np.array_equal(off, o2) and np.array_equal(idx, i2)
            assert np.array_equal(dist, d2)
    finally:
        ix.close()


def test_degenerate_thin_and_empty_inputs(pb):
    prm = pb.MlsParams(kernel=pb.KernelParams(0.1))
    iso = np.array([[0, 0, 0], [10, 0, 0], [10.01, 0, 0]], dtype=float)
    out, res = pb.smooth_cloud(iso, prm)
    assert (res.status == 3).all() and np.array_equal(out, iso)
    out, res = pb.smooth_cloud(np.zeros((0, 3)), prm)
    assert out.shape == (0, 3)
    line = np.c_[0.01 * np.arange(50), np.zeros(50), np.zeros(50)]
    out, res = pb.smooth_cloud(line, pb.MlsParams(kernel=pb.KernelParams(0.05)))
    assert (res.plane_status == 2).all() and (res.status == 3).all()
    with pytest.raises(pb.InvalidParam):
        pb.smooth_cloud(iso, pb.MlsParams(degree=0))


@pytest.mark.parametrize("n,h,deg", [(200, 0.05, 2), (500, 0.03, 3), (400, 0.05, 4)])
def test_sparse_clouds_degrade_like_the_oracle(pb, orc, n, h, deg):
    """Sparse random clouds: thin neighbourhoods step the degree down
    (DegradedDegree, mls.cpp:48-60) or pass the point through (Skipped,
    TooFewNeighbors); statuses, degrees used, plane statuses and iteration
    counts must be the oracle's, positions within rounding."""
    seen = np.zeros(4, dtype=int)
    for seed in range(4):
        P = np.random.default_rng(seed).uniform(-1, 1, (n, 3))
        out, res = pb.smooth_cloud(P, pb.MlsParams(kernel=pb.KernelParams(h), degree=deg))
        r = orc.mls_project(P, P, h, degree=deg)
        assert np.array_equal(res.status, r["status"])
        assert np.array_equal(res.degree_used, r["degree_used"])
        assert np.array_equal(res.plane_status, r["plane_status"])
        assert np.array_equal(res.iterations, r["iterations"])
        assert np.abs(out - r["projected"]).max() <= 1e-9
        skipped = res.status == 3
        assert np.array_equal(out[skipped], P[skipped])
        seen += np.bincount(res.status, minlength=4)
    assert seen[1] > 0 and seen[3] > 0, seen  # degraded and skipped points occur


@pytest.mark.parametrize("kind,n,seed,sigma,h,deg", CASES[:4])
def test_smooth_outcomes_equal_full_records(pb, kind, n, seed, sigma, h, deg):
    """pcs_mls_smooth_outcomes (queries = the index's own sorted points, 32 bytes
    per point back) against pcs_mls_smooth (312-byte records): the projected
    cloud is bit-identical and every outcome field equal; sparse clouds too."""
    for P in (cloud(pb, kind, n, seed, sigma),
              np.random.default_rng(seed).uniform(-1.0, 1.0, (300, 3))):
        prm = pb.MlsParams(kernel=pb.KernelParams(h), degree=deg)
        lean, ro = pb.smooth_cloud(P, prm)
        full, rf = pb.smooth_cloud(P, prm, full_records=True)
        assert np.array_equal(lean, full)
        assert np.array_equal(lean, ro.projected) and ro.coeffs is None
        for k in ("status", "degree_used", "iterations", "plane_status", "poly_status"):
            assert np.array_equal(getattr(ro, k), getattr(rf, k)), k


def test_smooth_without_records_buffer(pb):
    """pcs_mls_smooth with results == NULL (the call INTEGRATION.md shows) takes the
    two-launch path and returns the same cloud as the record path."""
    import ctypes as C
    from paper_2401_03365_b200 import _lib as L
    from paper_2401_03365_b200 import mls as M
    P = cloud(pb, "sphere", 3000, 11, 0.01)
    prm = pb.MlsParams(kernel=pb.KernelParams(0.2), degree=2)
    full, _ = pb.smooth_cloud(P, prm, full_records=True)
    out = np.zeros_like(P)
    d = M._desc(prm, -1)
    st = L.lib().pcs_mls_smooth(C.byref(d), P.ctypes.data_as(C.POINTER(C.c_double)), P.shape[0],
                                out.ctypes.data_as(C.POINTER(C.c_double)), None)
    assert st == 0 and np.array_equal(out, full)
    a, b = C.c_double(-1.0), C.c_double(-1.0)
    assert L.lib().pcs_mls_last_device_ms(C.byref(a), C.byref(b)) == 0
    assert a.value > 0.0 and b.value > 0.0


def test_center_bounds_equal_full_records(pb):
    """pcs_mls_smooth_bounds: the bounds of the query centres (plane iterates and
    frame origin) equal the full records' cmin / cmax bit for bit, on a dense and
    on a sparse cloud (skipped points keep their single centre)."""
    for P, h in ((cloud(pb, "torus", 3000, 5, 0.01), 0.1),
                 (np.random.default_rng(3).uniform(-1.0, 1.0, (300, 3)), 0.05)):
        prm = pb.MlsParams(kernel=pb.KernelParams(h), degree=2)
        lean, rb = pb.smooth_cloud(P, prm, center_bounds=True)
        full, rf = pb.smooth_cloud(P, prm, full_records=True)
        assert np.array_equal(lean, full)
        assert np.array_equal(rb.cmin, rf.cmin) and np.array_equal(rb.cmax, rf.cmax)
