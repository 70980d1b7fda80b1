"""The MLS oracle (oracle/lop_oracle.c orc_mls_project) pinned to the
reference's own MLS / WLS test properties (CPU, no GPU).

The reference's MLS cannot be built here (proj/src/wls.cpp needs Eigen, absent
from this image), so there are no golden vectors for this row: the oracle is
pinned by the analytic and property checks of proj/tests/test_wls.cpp and
test_mls.cpp, restated below, and by an independent dense weighted
least-squares solve (numpy) for the polynomial fit.  The host-only slab
partition of the product library (pcs_mls_partition) is checked here too.
"""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def O(orc):
    return orc


def plane_cloud(rng, n, sigma=0.0, extent=1.0):
    xy = rng.uniform(-extent, extent, (n, 2))
    z = rng.normal(0.0, sigma, n) if sigma > 0 else np.zeros(n)
    return np.c_[xy, z]


def theta(d, h):
    return np.exp(-(d / h) ** 2)


def test_exact_plane_frame_and_orientation(O):
    """test_wls.cpp:45-64: the frame converges onto the plane, normal toward r."""
    P = plane_cloud(np.random.default_rng(42), 50)
    r = O.mls_project(P, [[0, 0, 0.5], [0, 0, -0.5], [0.1, -0.2, 0.0]], 1.0, mode=O.MLS_PLANE)
    assert (r["plane_status"] == 0).all()
    assert np.allclose(r["normal"][0], [0, 0, 1], atol=1e-9)
    assert np.allclose(r["normal"][1], [0, 0, -1], atol=1e-9)
    assert np.abs(r["origin"][:2, 2]).max() < 1e-9
    assert r["normal"][2][2] > 0  # tie on the plane -> +z (test_wls.cpp:66-73)
    # orthonormal, right-handed frame (test_wls.cpp:75-94)
    for k in range(3):
        n, u, v = r["normal"][k], r["u"][k], r["v"][k]
        assert abs(np.dot(u, v)) < 1e-12 and abs(np.dot(u, n)) < 1e-12
        assert np.allclose(np.cross(u, v), n, atol=1e-12)


def test_thin_and_degenerate_neighbourhoods(O):
    """test_wls.cpp:203-215."""
    r = O.mls_project([[0, 0, 0], [0.1, 0, 0]], [[0, 0, 0.1]], 1.0, mode=O.MLS_PLANE)
    assert r["plane_status"][0] == 1  # TooFewNeighbors
    line = np.c_[0.1 * np.arange(10), np.zeros(10), np.zeros(10)]
    r = O.mls_project(line, [[0.45, 0.05, 0.0]], 1.0, mode=O.MLS_PLANE)
    assert r["plane_status"][0] == 2  # DegenerateNeighborhood


def test_single_pass_no_convergence(O):
    """test_wls.cpp:217-224: max_iter = 1 -> NoConvergence, a usable frame."""
    P = plane_cloud(np.random.default_rng(48), 100, 0.05)
    r = O.mls_project(P, [[0, 0, 0.2]], 0.7, max_iter=1, mode=O.MLS_PLANE)
    assert r["plane_status"][0] == 3 and r["iterations"][0] == 1
    assert abs(np.linalg.norm(r["normal"][0]) - 1.0) < 1e-12


def frame_z(origin=(0, 0, 0)):
    return np.array(list(origin) + [0, 0, 1, 1, 0, 0, 0, 1, 0], dtype=np.float64)


def test_polynomial_exact_plane_and_paraboloid(O):
    """test_wls.cpp:226-268."""
    P = plane_cloud(np.random.default_rng(49), 60, 0.0, 0.5)
    for deg in range(1, 5):
        r = O.mls_project(P, [[0, 0, 0]], 1.0, degree=deg, mode=O.MLS_POLY, frames=frame_z())
        assert r["poly_status"][0] == 0
        assert np.abs(r["coeffs"][0]).max() < 1e-10
    rng = np.random.default_rng(50)
    xy = rng.uniform(-0.5, 0.5, (80, 2))
    Q = np.c_[xy, xy[:, 0] ** 2 + xy[:, 1] ** 2]
    r = O.mls_project(Q, [[0, 0, 0]], 1.0, degree=2, mode=O.MLS_POLY, frames=frame_z())
    assert np.allclose(r["coeffs"][0][:6], [0, 0, 0, 1, 0, 1], atol=1e-8)


def basis(u, v, deg):
    return np.stack([u ** a * v ** (s - a) for s in range(deg + 1) for a in range(s, -1, -1)], -1)


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_polynomial_matches_dense_weighted_least_squares(O, deg):
    """test_wls.cpp:270-306 restated: the fit equals the dense weighted
    normal-equation solution (independent numpy solve)."""
    rng = np.random.default_rng(51 + deg)
    for trial in range(10):
        P = rng.uniform(-0.8, 0.8, (40, 3))
        o = rng.uniform(-0.05, 0.05, 3)
        A, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        u, v, n = A[:, 0], A[:, 1], np.cross(A[:, 0], A[:, 1])
        fr = np.r_[o, n, u, v]
        r = O.mls_project(P, [o], 1.0, degree=deg, mode=O.MLS_POLY, frames=fr)
        assert r["poly_status"][0] == 0
        d = P - o
        B = basis(d @ u, d @ v, deg)
        w = theta(np.linalg.norm(d, axis=1), 1.0) * (np.linalg.norm(d, axis=1) <= 3.0)
        M = B.T @ (w[:, None] * B)
        b = B.T @ (w * (d @ n))
        want = np.linalg.solve(M, b)
        K = want.size
        assert np.allclose(r["coeffs"][0][:K], want, rtol=0, atol=1e-10 * (1 + np.abs(want).max()))


def test_polynomial_failure_modes(O):
    """test_wls.cpp:340-361."""
    five = np.array([[0.1 * i, 0.05 * ((i * 7) % 5), 0.0] for i in range(5)])
    fr = frame_z((0.2, 0.1, 0.0))
    assert O.mls_project(five, [[0.2, 0.1, 0]], 1.0, degree=2, mode=O.MLS_POLY, frames=fr)["poly_status"][0] == 1
    assert O.mls_project(five, [[0.2, 0.1, 0]], 1.0, degree=1, mode=O.MLS_POLY, frames=fr)["poly_status"][0] == 0
    stack = np.c_[np.zeros(10), np.zeros(10), 0.01 * np.arange(10)]
    assert O.mls_project(stack, [[0.2, 0.1, 0]], 1.0, degree=1, mode=O.MLS_POLY, frames=fr)["poly_status"][0] == 2


def test_projection_contracts(O):
    """test_mls.cpp:43-61, 77-100, 150-156: plane projection, fixed points,
    Skipped pass-through."""
    P = plane_cloud(np.random.default_rng(71), 300)
    r = O.mls_project(P, [[0.2, -0.1, 0.7], [0.2, -0.1, 0.0]], 1.0)
    assert (r["status"] == 0).all()
    assert np.allclose(r["projected"], [[0.2, -0.1, 0.0]] * 2, atol=1e-9)
    iso = np.array([[0, 0, 0], [10, 0, 0], [10.01, 0, 0]], dtype=float)
    r = O.mls_project(iso, iso, 0.1)
    assert (r["status"] == 3).all() and np.array_equal(r["projected"], iso)


def test_smoothing_reduces_noise_on_sphere(pb, O):
    """test_mls.cpp:102-111 on the oracle: radial RMS error drops."""
    clean = pb.generate_surface("sphere", 2000, 19)
    noisy = pb.add_noise(clean, 0.05, 20)
    r = O.mls_project(noisy, noisy, 0.25)
    assert (r["status"] != 3).all()
    rms = lambda X: np.sqrt(np.mean((np.linalg.norm(X, axis=1) - 1.0) ** 2))  # noqa: E731
    assert rms(r["projected"]) < rms(noisy)


# ---- host-only slab partition of the product library (proj/src/parallel.cpp:64-127)
def test_partition_collinear_cuts(pb):
    """test_parallel.cpp:43-57."""
    P = np.c_[np.arange(8.0), np.zeros(8), np.zeros(8)]
    axis, cuts, wof = pb.partition(P, 4, 0.5)
    assert axis == 0 and list(cuts) == [1.5, 3.5, 5.5]
    assert np.bincount(wof).tolist() == [2, 2, 2, 2]


def test_partition_balanced_multiset(pb):
    """test_parallel.cpp:59-80 and 89-97 (more workers than points)."""
    rng = np.random.default_rng(82)
    P = rng.uniform(-1, 1, (10000, 3))
    axis, cuts, wof = pb.partition(P, 4, 0.3)
    cnt = np.bincount(wof, minlength=4)
    assert cnt.max() - cnt.min() <= 1 and cnt.max() == 2500
    c = P[:, axis]
    for u in range(4):  # equal-count slabs in axis order, ties by index
        lo = -np.inf if u == 0 else cuts[u - 1]
        hi = np.inf if u == 3 else cuts[u]
        assert ((c[wof == u] >= lo) & (c[wof == u] <= hi)).all()
    axis, cuts, wof = pb.partition([[0, 0, 0], [1, 0, 0], [2, 0, 0]], 5, 0.5)
    assert np.bincount(wof, minlength=5).tolist() == [1, 1, 1, 0, 0]


def test_partition_rejects_bad_arguments(pb):
    """test_parallel.cpp:82-87."""
    P = np.random.default_rng(83).uniform(-1, 1, (10, 3))
    with pytest.raises(pb.InvalidParam):
        pb.partition(P, 0, 0.5)
    with pytest.raises(pb.EmptyCloud):
        pb.partition(np.zeros((0, 3)), 2, 0.5)
    with pytest.raises(pb.InvalidParam):
        pb.partition(P, 2, 0.0)


def test_mls_params_validation(pb):
    """MlsParams::validate (proj/include/pcs/mls.hpp:20-29)."""
    for bad in (pb.MlsParams(kernel=pb.KernelParams(0.0)), pb.MlsParams(degree=5),
                pb.MlsParams(plane_tol=0.0), pb.MlsParams(plane_max_iter=0)):
        with pytest.raises(pb.InvalidParam):
            bad.validate()
