"""Pins the CPU restatement of the deviation metrics (oracle/lop_oracle.c:
nearest, deviation, point_triangle_distance, deviation_to_mesh) before it is
used as the checker of the B200 kernels (tests/test_gpu_metrics.py):

* bit-for-bit against tests/golden/reference_metrics.npz, produced by the
  unmodified reference (tests/golden/make_golden_metrics.py),
* bit-for-bit against the live reference build (oracle/_ref) when present,
* the error contract of proj/src/metrics.cpp (empty cloud, then empty reference).
"""
import numpy as np
import pytest


def test_nearest_bit_exact_vs_reference_fixture(orc, golden_metrics):
    g = golden_metrics
    for k in ("", "_lattice"):
        idx, dist = orc.nearest_all(g[f"nn{k}_C"], g[f"nn{k}_Q"])
        assert np.array_equal(idx, g[f"nn{k}_idx"])
        assert np.array_equal(dist, g[f"nn{k}_dist"])


def test_deviation_bit_exact_vs_reference_fixture(orc, golden_metrics):
    g = golden_metrics
    rep, dist = orc.deviation(g["dev_cloud"], g["dev_ref"])
    assert np.array_equal(rep, g["dev_report"])
    assert np.array_equal(dist, g["dev_dist"])


def test_mesh_bit_exact_vs_reference_fixture(orc, golden_metrics):
    g = golden_metrics
    rep, dist = orc.deviation_to_mesh(g["mesh_P"], g["mesh_T"])
    assert np.array_equal(rep, g["mesh_report"])
    assert np.array_equal(dist, g["mesh_dist"])
    ptri = [orc.point_triangle_distance(p, g["mesh_T"][t % 80])
            for t, p in enumerate(g["mesh_P"][:200])]
    assert np.array_equal(np.array(ptri), g["ptri"])


def test_point_triangle_fixed_cases(orc):
    # proj/tests/test_metrics.cpp:110-119 (face, vertex, edge regions)
    tri = [0, 0, 0, 4, 0, 0, 0, 4, 0]
    assert orc.point_triangle_distance([1, 1, 0], tri) == 0.0
    assert orc.point_triangle_distance([1, 1, 0.7], tri) == pytest.approx(0.7, rel=1e-15)
    assert orc.point_triangle_distance([-3, 0, 0], tri) == pytest.approx(3.0, rel=1e-15)
    assert orc.point_triangle_distance([2, -1, 0], tri) == pytest.approx(1.0, rel=1e-15)
    assert orc.point_triangle_distance([5, 5, 0], tri) == pytest.approx(3 * 2 ** 0.5, rel=1e-12)


def test_metrics_vs_live_reference(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built here")
    rng = np.random.default_rng(7)
    for trial in range(3):
        C = rng.uniform(-1, 1, (2000, 3))
        C[500:550] = C[:50]
        Q = np.concatenate([rng.uniform(-1.3, 1.3, (700, 3)), C[:50]])
        i1, d1 = orc.nearest_all(C, Q)
        i2, d2 = orc.ref_nearest_all(C, Q)
        assert np.array_equal(i1, i2) and np.array_equal(d1, d2)
        r1, _ = orc.deviation(Q, C)
        r2, _ = orc.ref_deviation(Q, C)
        assert np.array_equal(r1, r2)
        T = rng.uniform(-1, 1, (40, 9))
        T[0, 6:9] = T[0, 3:6]
        m1, _ = orc.deviation_to_mesh(Q[:300], T)
        m2, _ = orc.ref_deviation_to_mesh(Q[:300], T)
        assert np.array_equal(m1, m2)


def test_metrics_error_contract(orc):
    one = np.zeros((1, 3))
    with pytest.raises(orc.OracleError):
        orc.deviation(np.zeros((0, 3)), one)
    with pytest.raises(orc.OracleError):
        orc.deviation(one, np.zeros((0, 3)))
    with pytest.raises(orc.OracleError):
        orc.deviation_to_mesh(one, np.zeros((0, 9)))
