"""Parity of the B200 deviation metrics (csrc/nn.cu) with the reference.

Bit-exact: nearest indices (smallest index among equal squared distances) and
distances, the aggregated reports (index-order sums, as proj/src/metrics.cpp:
11-37) and the mesh distances — against the reference fixture
(tests/golden/reference_metrics.npz), the CPU restatement (oracle/) and, at
config-3 scale, the reference kd-tree itself (oracle/_ref) when it was built.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nearest_bit_exact_vs_reference_fixture(pb, golden_metrics):
    g = golden_metrics
    for k in ("", "_lattice"):
        idx, dist = pb.nearest_all(g[f"nn{k}_C"], g[f"nn{k}_Q"], device=0)
        assert np.array_equal(idx, g[f"nn{k}_idx"]), k
        assert np.array_equal(dist, g[f"nn{k}_dist"]), k


def test_deviation_and_mesh_bit_exact_vs_reference_fixture(pb, golden_metrics):
    g = golden_metrics
    r = pb.deviation(g["dev_cloud"], g["dev_ref"], keep_distances=True, device=0)
    assert [r.n, r.mean_distance, r.std_deviation, r.max_distance] == list(g["dev_report"])
    assert np.array_equal(r.distances, g["dev_dist"])
    r = pb.deviation_to_mesh(g["mesh_P"], g["mesh_T"].reshape(-1, 3, 3), keep_distances=True,
                             device=0)
    assert [r.n, r.mean_distance, r.std_deviation, r.max_distance] == list(g["mesh_report"])
    assert np.array_equal(r.distances, g["mesh_dist"])


@pytest.mark.parametrize("case", ["uniform", "duplicates", "far_queries", "single_point",
                                  "planar", "coincident_queries"])
def test_nearest_edge_cases_vs_oracle(pb, orc, case):
    rng = np.random.default_rng(11)
    C = rng.uniform(-1, 1, (5000, 3))
    Q = rng.uniform(-1.1, 1.1, (3000, 3))
    if case == "duplicates":
        C[2500:] = C[:2500]                       # every point twice: index tie-break
    elif case == "far_queries":
        Q = rng.uniform(-1e3, 1e3, (500, 3))
    elif case == "single_point":
        C = C[:1]
    elif case == "planar":
        C[:, 2] = 0.25                            # zero extent along z
        Q[:, 2] = rng.choice([0.25, 0.0, 1.0], Q.shape[0])
    elif case == "coincident_queries":
        Q = C[rng.integers(0, C.shape[0], 2000)]  # d = 0 hits
    i1, d1 = pb.nearest_all(C, Q, device=0)
    i2, d2 = orc.nearest_all(C, Q)
    assert np.array_equal(i1, i2)
    assert np.array_equal(d1, d2)


def test_deviation_vs_oracle_and_error_contract(pb, orc):
    rng = np.random.default_rng(12)
    R = rng.normal(size=(20000, 3))
    X = rng.normal(size=(4000, 3))
    r = pb.deviation(X, R, keep_distances=True, device=0)
    o, od = orc.deviation(X, R)
    assert [r.n, r.mean_distance, r.std_deviation, r.max_distance] == list(o)
    assert np.array_equal(r.distances, od)
    assert r.std_deviation >= r.mean_distance * (1 - 1e-12)
    with pytest.raises(pb.EmptyCloud, match="cloud is empty"):
        pb.deviation(np.zeros((0, 3)), R, device=0)
    with pytest.raises(pb.EmptyCloud, match="reference cloud is empty"):
        pb.deviation(X, np.zeros((0, 3)), device=0)
    with pytest.raises(pb.EmptyMesh):
        pb.deviation_to_mesh(X, np.zeros((0, 3, 3)), device=0)
    with pytest.raises(pb.EmptyCloud):
        pb.deviation_to_mesh(np.zeros((0, 3)), np.zeros((1, 3, 3)), device=0)
    with pytest.raises(pb.EmptyCloud):
        pb.nearest_all(np.zeros((0, 3)), X, device=0)


def test_mesh_vs_oracle_with_degenerate_triangles(pb, orc):
    rng = np.random.default_rng(13)
    T = rng.uniform(-1, 1, (300, 9))
    T[::17, 6:9] = T[::17, 0:3]                   # repeated vertex
    T[::23, 3:6] = T[::23, 0:3]
    T[::23, 6:9] = T[::23, 0:3]                   # point triangle
    T[::29, 6:9] = 0.25 * T[::29, 0:3] + 0.75 * T[::29, 3:6]  # collinear
    P = rng.uniform(-1.5, 1.5, (3000, 3))
    r = pb.deviation_to_mesh(P, T.reshape(-1, 3, 3), keep_distances=True, device=0)
    o, od = orc.deviation_to_mesh(P, T)
    assert np.array_equal(r.distances, od)
    assert [r.n, r.mean_distance, r.std_deviation, r.max_distance] == list(o)


def test_deviation_config3_scale_vs_reference_kdtree(pb, orc):
    """A projected-set-sized query cloud against the config-3 data (30% scale:
    P = 3M, X0 = 300K): every nearest index and distance equals the reference's
    own kd-tree result (oracle/_ref, all host cores)."""
    if not orc.ref_available():
        pytest.skip("oracle/_ref not present")
    P, X0 = pb.generate_config(3, 0.3)
    rng = np.random.default_rng(14)
    Q = X0 + rng.normal(scale=0.002, size=X0.shape)
    i1, d1 = pb.nearest_all(P, Q, device=0)
    i2, d2 = orc.ref_nearest_all(P, Q)
    assert np.array_equal(i1, i2)
    assert np.array_equal(d1, d2)
