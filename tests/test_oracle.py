"""Pins the CPU oracle (oracle/lop_oracle.c) before it is trusted as the checker.

* against the reference's own golden values (test_noise.cpp:64-72 KAT,
  test_lop.cpp:119-133 frozen ratio),
* bit-for-bit against the committed fixture produced by the unmodified
  reference (tests/golden/make_golden.py),
* bit-for-bit against the live reference build (oracle/_ref) on fresh random
  instances, when it is present,
* and the two variants the reference lacks (eta = -r, WLOP) by properties.
"""
import numpy as np
import pytest

from conftest import bbox_diag


def test_rng_kat_matches_reference_golden(orc):
    # proj/tests/test_noise.cpp:64-72: first Box-Muller normals of mt19937_64(1)
    out = orc.add_noise(np.zeros((1, 3)), 1.0, 1)[0]
    assert out[0] == pytest.approx(1.312851528985562, rel=1e-13)
    assert out[1] == pytest.approx(1.5159465040060625, rel=1e-13)
    assert out[2] == pytest.approx(1.2506039211781217, rel=1e-13)


def test_generators_and_noise_bit_exact(orc, golden):
    assert np.array_equal(orc.plane(100, 7), golden["surface_0"])
    assert np.array_equal(orc.sphere(100, 7), golden["surface_1"])
    assert np.array_equal(orc.add_noise(golden["noise_in"], 0.1, 9), golden["noise_out"])


def test_frozen_plane_ratio(orc):
    # proj/tests/test_lop.cpp:119-133 (also acceptance.cpp:390-409)
    D = orc.add_noise(orc.plane(2000, 11), 0.05, 55)
    init = D[::10][:200]
    r = orc.lop_project(D, init, 0.3, 3.0, 0.4, 30)
    before = np.abs(init[:, 2]).sum() / 200
    after = np.abs(r.points[:, 2]).sum() / 200
    assert after < before
    assert after / before == pytest.approx(0.07335543385137086, rel=0.05)
    # the reference reproduces this value to the last digits with this toolchain
    assert abs(after / before - 0.07335543385137086) < 1e-15


@pytest.mark.parametrize("name", ["plane", "single", "pair", "isolated", "coincident", "random",
                                  "sphere", "duplicates"])
def test_lop_bit_exact_vs_reference_fixture(orc, golden, name):
    P = golden[f"lop_{name}_P"]
    X0 = golden[f"lop_{name}_X0"]
    h, cut, mu, it = golden[f"lop_{name}_params"]
    r = orc.lop_project(P, X0, h, cut, mu, int(it))
    assert np.array_equal(r.points, golden[f"lop_{name}_out"])
    s = golden[f"lop_{name}_summary"]
    assert (r.iterations_run, int(r.converged), r.isolated_events, r.coincident_pairs) == tuple(s)
    assert np.array_equal(np.asarray(r.isolated_indices, dtype=np.int64),
                          golden[f"lop_{name}_isolated"])


def test_radius_query_bit_exact_vs_reference_fixture(orc, golden):
    off, idx, dist = orc.radius_query_all(golden["rq_cloud"], golden["rq_queries"],
                                          float(golden["rq_r"]))
    assert np.array_equal(off, golden["rq_offsets"])
    assert np.array_equal(idx, golden["rq_idx"])
    assert np.array_equal(dist, golden["rq_dist"])


def test_oracle_vs_live_reference(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built on this host (fixture test covers it)")
    rng = np.random.default_rng(2024)
    for trial in range(4):
        P = rng.uniform(-1, 1, (400, 3))
        X0 = np.concatenate([P[rng.choice(400, 30, replace=False)], rng.uniform(-1, 1, (10, 3))])
        h = [0.1, 0.15, 0.2, 0.3][trial]
        a = orc.lop_project(P, X0, h, 3.0, 0.35, 8)
        b = orc.ref_lop_project(P, X0, h, 3.0, 0.35, 8)
        assert np.array_equal(a.points, b.points)
        assert (a.iterations_run, a.isolated_events, a.coincident_pairs) == \
               (b.iterations_run, b.isolated_events, b.coincident_pairs)
        o1, i1, d1 = orc.radius_query_all(P, X0, 2 * h)
        o2, i2, d2 = orc.ref_radius_query_all(P, X0, 2 * h)
        assert np.array_equal(o1, o2) and np.array_equal(i1, i2) and np.array_equal(d1, d2)


def test_validation_order(orc):
    P = np.zeros((1, 3))
    with pytest.raises(orc.OracleError) as e:
        orc.lop_project(P, P, 0.0, 3.0, 0.0, 1)
    assert e.value.kind == "InvalidParam"
    with pytest.raises(orc.OracleError) as e:
        orc.lop_project(np.zeros((0, 3)), P, 1.0, 3.0, 0.0, 1)
    assert e.value.kind == "EmptyCloud"
    r = orc.lop_project(P, np.zeros((0, 3)), 1.0, 3.0, 0.0, 1)
    assert r.points.shape == (0, 3) and r.iterations_run == 0


def test_neg_linear_and_wlop_properties(orc):
    # no reference implementation exists: pin the restatement by properties
    rng = np.random.default_rng(7)
    P = rng.uniform(-1, 1, (300, 3))
    X0 = P[rng.choice(300, 25, replace=False)]
    shift = np.array([3.5, -1.25, 0.75])
    for eta in (orc.ETA_INV_CUBE, orc.ETA_NEG_LINEAR):
        for wlop in (False, True):
            a = orc.lop_project(P, X0, 0.15, 3.0, 0.3, 6, eta=eta, wlop=wlop)
            b = orc.lop_project(P + shift, X0 + shift, 0.15, 3.0, 0.3, 6, eta=eta, wlop=wlop)
            assert np.abs(b.points - shift - a.points).max() < 1e-9 * bbox_diag(P)
    # mu = 0: eta and the projected-set density play no role
    a = orc.lop_project(P, X0, 0.15, 3.0, 0.0, 4, eta=orc.ETA_NEG_LINEAR)
    b = orc.lop_project(P, X0, 0.15, 3.0, 0.0, 4, eta=orc.ETA_INV_CUBE)
    assert np.array_equal(a.points, b.points)
    # density weight of a lattice corner: 3 axis neighbours at 0.1 and 3 face
    # diagonals at 0.1*sqrt(2) lie inside the support 0.15
    g = np.stack(np.meshgrid(*[np.arange(8) * 0.1] * 3, indexing="ij"), -1).reshape(-1, 3)
    v = orc.density_weights(g, 0.05, 3.0)
    assert v.min() >= 1.0
    corner = 1.0 + 3 * orc.theta(0.1, 0.05, 3.0) + 3 * orc.theta(np.sqrt(0.02), 0.05, 3.0)
    assert v[0] == pytest.approx(corner, rel=1e-14)


def test_density_weights_count_coincident_duplicates(orc):
    C = np.array([[0.0, 0, 0], [0.0, 0, 0], [1.0, 0, 0]])
    v = orc.density_weights(C, 0.2, 3.0)  # support 0.6: the far point is alone
    assert v[0] == 2.0 and v[1] == 2.0 and v[2] == 1.0  # theta(0) = 1 for the duplicate


# ----------------------------------------------------------------------------
# eta = -r: pinned to the reference's own lop.cpp (|eta'| bound to 1 at link
# time, oracle/ref_etar_wrap.cpp) — fixture and live build
# ----------------------------------------------------------------------------
ETAR = ["height", "sphere", "duplicates", "random_isolated"]


@pytest.fixture(scope="module")
def golden_etar():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_etar.npz"))


@pytest.mark.parametrize("name", ETAR)
def test_neg_linear_bit_exact_vs_reference_fixture(orc, golden_etar, name):
    g = golden_etar
    h, cut, mu, it = g[f"lop_{name}_params"]
    r = orc.lop_project(g[f"lop_{name}_P"], g[f"lop_{name}_X0"], h, cut, mu, int(it),
                        eta=orc.ETA_NEG_LINEAR)
    assert np.array_equal(r.points, g[f"lop_{name}_out"])
    assert (r.iterations_run, int(r.converged), r.isolated_events, r.coincident_pairs) == \
        tuple(g[f"lop_{name}_summary"])
    assert np.array_equal(np.asarray(r.isolated_indices, dtype=np.int64),
                          g[f"lop_{name}_isolated"])
    if name == "duplicates":
        assert r.coincident_pairs > 0
    if name == "random_isolated":
        assert r.isolated_events > 0


def test_neg_linear_bit_exact_vs_live_reference(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(77)
    for k in range(3):
        P = rng.uniform(-1, 1, (800, 3))
        X0 = np.concatenate([P[rng.choice(800, 60, replace=False)], P[:3]])  # coincident pairs
        a = orc.lop_project(P, X0, 0.1, 4.0, 0.45, 5, eta=orc.ETA_NEG_LINEAR)
        b = orc.ref_lop_project(P, X0, 0.1, 4.0, 0.45, 5, eta=orc.ETA_NEG_LINEAR)
        assert np.array_equal(a.points, b.points)
        assert (a.isolated_events, a.coincident_pairs) == (b.isolated_events, b.coincident_pairs)
        # and the wrap really changed eta: the shipped eta = 1/(3r^3) differs
        c = orc.ref_lop_project(P, X0, 0.1, 4.0, 0.45, 5)
        assert np.abs(c.points - b.points).max() > 1e-6


@pytest.mark.parametrize("cfg,scale", [(1, 0.1), (2, 0.01), (3, 0.002), (4, 0.003), (5, 0.0005)])
def test_oracle_config_generator_matches_product(orc, pb, cfg, scale):
    """The oracle's restated config generator (used by bench.py's reference arm
    so that it never loads the product library) draws exactly what the
    product's host generator draws (host code, no device needed)."""
    P, X0 = orc.generate_config(cfg, scale)
    P2, X2 = pb.generate_config(cfg, scale)
    assert np.array_equal(P, P2) and np.array_equal(X0, X2)


def test_sweep_rows_matches_full_sweep(orc):
    rng = np.random.default_rng(3)
    P = rng.uniform(-1, 1, (6000, 3)) * np.array([1, 1, 0.05])
    X = np.concatenate([P[rng.choice(6000, 600, replace=False)], P[:2], [[9.0, 9.0, 9.0]]])
    rows = np.array([0, 5, 600, 601, 602, 77], dtype=np.uint32)
    for eta in (orc.ETA_INV_CUBE, orc.ETA_NEG_LINEAR):
        for wlop in (False, True):
            full, iso, co, _ = orc.lop_sweep(P, X, 0.08, 3.0, 0.45, eta=eta, wlop=wlop)
            nxt, cnt = orc.lop_sweep_rows(P, X, rows, 0.08, 3.0, 0.45, eta=eta, wlop=wlop)
            assert np.abs(nxt - full[rows]).max() <= 1e-15
            assert np.array_equal(cnt[:, 2], co[rows])
            assert np.array_equal(cnt[:, 3] & 1, iso[rows])
    r = orc.lop_project(P, X, 0.08, 3.0, 0.45, 1, eta=orc.ETA_NEG_LINEAR)
    _, cnt = orc.lop_sweep_rows(P, X, np.arange(X.shape[0]), 0.08, 3.0, 0.45,
                                eta=orc.ETA_NEG_LINEAR)
    assert (cnt[:, 0].sum(), cnt[:, 1].sum()) == (r.interactions_attr, r.interactions_rep)
    assert cnt[602, 3] == 1  # the far point is isolated
