"""Parity of the B200 path against the oracle and the reference fixtures (GPU).

Every call goes through the C ABI (include/pcs_lop.h) via the Python mirror.
Bars (north star): neighbour lists and sort order bit-exact; positions within
1e-5 x bounding-box diagonal.  fp32 runs are compared with the oracle run on
the same fp32-rounded inputs; for multi-sweep fp32 trajectories the oracle
stores its iterate in fp32 too (oracle store_f32), mirroring fp32 storage.
"""
import numpy as np
import pytest

from conftest import bbox_diag

pytestmark = pytest.mark.gpu

F32 = np.float32


def r32(a):
    return np.asarray(a, dtype=F32).astype(np.float64)


# ----------------------------------------------------------------------------
# reference fixtures (tests/golden/reference_cases.npz, produced by the reference)
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["plane", "single", "pair", "isolated", "coincident", "random",
                                  "sphere", "duplicates"])
def test_fp64_matches_reference_fixture(pb, golden, name):
    P = golden[f"lop_{name}_P"]
    X0 = golden[f"lop_{name}_X0"]
    h, cut, mu, it = golden[f"lop_{name}_params"]
    prm = pb.LopParams(kernel=pb.KernelParams(h, cut), mu=mu, iterations=int(it))
    out, s = pb.lop_project(P, X0, prm, precision="fp64")
    ref = golden[f"lop_{name}_out"]
    tol = 1e-9 * max(bbox_diag(np.concatenate([P, X0])), 1.0)
    assert np.abs(out - ref).max() <= tol
    it_run, conv, iso_ev, coinc = golden[f"lop_{name}_summary"]
    assert (s.iterations_run, int(s.converged), s.isolated_events, s.coincident_pairs) == \
           (it_run, conv, iso_ev, coinc)
    assert s.isolated_indices == list(golden[f"lop_{name}_isolated"])


def test_radius_queries_match_reference_fixture(pb, golden):
    off, idx = pb.radius_query_all(golden["rq_cloud"], golden["rq_queries"], float(golden["rq_r"]))
    assert np.array_equal(off, golden["rq_offsets"])
    assert np.array_equal(idx, golden["rq_idx"])


# ----------------------------------------------------------------------------
# the reference's LOP unit tests (proj/tests/test_lop.cpp:52-176), restated
# ----------------------------------------------------------------------------
def mk(pb, h, mu, it=30):
    return pb.LopParams(kernel=pb.KernelParams(h), mu=mu, iterations=it)


def test_single_point_absorbs(pb):
    data = np.array([[0.3, -0.2, 0.8]])
    q, s = pb.lop_project(data, np.array([[0.5, 0.1, 0.6]]), mk(pb, 1.0, 0.0))
    assert np.linalg.norm(q[0] - data[0]) < 1e-12 and s.converged


def test_isolated_and_coincident(pb):
    q, s = pb.lop_project(np.zeros((1, 3)), np.array([[5.0, 0, 0]]), mk(pb, 0.1, 0.0))
    assert np.array_equal(q[0], [5.0, 0, 0]) and s.isolated_events >= 1
    assert s.isolated_indices == [0]
    q, s = pb.lop_project(np.array([[1.0, 2, 3]]), np.array([[1.0, 2, 3]]), mk(pb, 0.5, 0.0))
    assert np.array_equal(q[0], [1, 2, 3]) and s.converged and s.isolated_events == 0


def test_translation_equivariance(pb):
    rng = np.random.default_rng(142)
    data = rng.uniform(-1, 1, (100, 3))
    init = rng.uniform(-0.5, 0.5, (10, 3))
    shift = np.array([3.5, -1.25, 0.75])
    for prec, tol in (("fp64", 1e-9), ("fp32", 1e-5)):
        q, _ = pb.lop_project(data, init, mk(pb, 0.6, 0.3, 10), precision=prec)
        qs, _ = pb.lop_project(data + shift, init + shift, mk(pb, 0.6, 0.3, 10), precision=prec)
        assert np.abs(qs - (q + shift)).max() < tol


def test_descent_mu0(pb, orc):
    # one mu = 0 sweep never increases the frozen-weight attraction objective
    rng = np.random.default_rng(141)
    for _ in range(20):
        data = rng.uniform(-1, 1, (60, 3))
        init = rng.uniform(-0.8, 0.8, (8, 3))
        nxt, _ = pb.lop_project(data, init, mk(pb, 0.8, 0.0, 1))
        for i in range(8):
            d0 = np.linalg.norm(data - init[i], axis=1)
            w = np.array([orc.theta(d, 0.8, 3.0) for d in d0])
            before = (d0 * w).sum()
            after = (np.linalg.norm(data - nxt[i], axis=1) * w).sum()
            if before > 0:
                assert after <= before * (1 + 1e-12)


# ----------------------------------------------------------------------------
# configuration 1 (fp64, full size) against the oracle
# ----------------------------------------------------------------------------
def test_config1_full_fp64(pb, orc):
    P, X0 = pb.generate_config(1)
    prm, c = pb.config_params(1)
    out, s = pb.lop_project(P, X0, prm, precision="fp64")
    r = orc.lop_project(P, X0, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu, prm.iterations)
    # fp64 on both sides; only the summation order differs (lane-strided partial
    # sums vs index order), amplified over 20 sweeps to ~1e-7 here
    assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)
    assert (s.iterations_run, s.converged, s.isolated_events, s.coincident_pairs) == \
           (r.iterations_run, r.converged, r.isolated_events, r.coincident_pairs)
    assert (s.interactions_attr, s.interactions_rep) == (r.interactions_attr, r.interactions_rep)


# ----------------------------------------------------------------------------
# fp32 fused kernel: one sweep from the same state must be exact in its
# neighbour sets and within a few fp32 ulps in position (configs 2-5, scaled)
# ----------------------------------------------------------------------------
SCALED = [(2, 0.02, 0.3), (3, 0.01, 0.2), (4, 0.01, 0.3), (5, 0.001, 0.3)]


def scaled_case(pb, cfg, scale, h):
    P, X0 = pb.generate_config(cfg, scale)
    prm, c = pb.config_params(cfg, h=h)
    return r32(P), r32(X0), prm, c


@pytest.mark.parametrize("cfg,scale,h", SCALED)
@pytest.mark.parametrize("start", [0, 12])
def test_fp32_single_sweep_exact_neighbours(pb, orc, cfg, scale, h, start):
    P, X0, prm, c = scaled_case(pb, cfg, scale, h)
    eta = orc.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else orc.ETA_INV_CUBE
    X = X0
    if start:
        prm.iterations = start
        X, _ = pb.lop_project(P, X0, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    prm.iterations = 1
    out, s = pb.lop_project(P, X, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    r = orc.lop_project(P, X, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu, 1, eta=eta,
                        wlop=c["wlop"], store_f32=True)
    # identical neighbour sets => identical interaction counts
    assert (s.interactions_attr, s.interactions_rep) == (r.interactions_attr, r.interactions_rep)
    assert (s.isolated_events, s.coincident_pairs) == (r.isolated_events, r.coincident_pairs)
    ext = np.abs(P).max()
    assert np.abs(out - r.points).max() <= 4 * np.finfo(F32).eps * ext


@pytest.mark.parametrize("cfg,scale,h,its", [(3, 0.01, 0.2, 15), (5, 0.001, 0.3, 10),
                                             (4, 0.01, 0.3, 20), (2, 0.02, 0.3, 30)])
def test_fp32_full_trajectory(pb, orc, cfg, scale, h, its):
    """Full iteration count, bar 1e-5 x bbox diagonal, in two parts.

    (1) Shadowing: EVERY sweep of the B200 run is the reference's map applied to
    the B200's own state — per query, identical attraction / repulsion /
    coincident counts and flags, and the new position within 4 fp32 ulps
    (orc_lop_sweep_rows, i.e. lop.cpp:41-100 on spatial.cpp:82-111).

    (2) End state against the oracle's own fp32 trajectory.  LOP/WLOP with
    eta = -r is chaotic on configs 2 and 4: the oracle started from its own
    sweep-1 state perturbed by ONE fp32 ulp ends 30/20 sweeps later beyond the
    bar on ~1.5% of the points (measured: config 4 52/4000, config 2 31/2000;
    no zero-distance or anchor event involved).  So a point beyond the bar must
    be (a) a point whose 1-ulp perturbation the reference itself amplifies to
    >= tol/100 in one of three perturbed oracle trajectories (a "sensitive"
    point, ~10-20% of configs 2/4, none of configs 3/5), or (b) at or within one
    support of a discontinuity of lop.cpp:55-69 (zero-distance sample, anchor)
    met in either run.  Any other outlier fails; configs 3 and 5 must meet the
    bar on every point."""
    P, X0, prm, c = scaled_case(pb, cfg, scale, h)
    prm.iterations = its
    eta = orc.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else orc.ETA_INV_CUBE
    kw = dict(eta=eta, wlop=c["wlop"])
    h4, mu = prm.kernel.h, prm.mu
    ext = float(np.abs(P).max())
    eps = float(np.finfo(F32).eps)
    rows = np.arange(X0.shape[0], dtype=np.uint32)
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    try:
        plan.upload(P, X0)
        plan.record_counts(True)
        X = X0
        worst = 0.0
        for k in range(its):
            plan.run(1)
            Xn, _ = plan.download()
            cnt, gpu_ever = plan.query_counts()
            nxt, oc = orc.lop_sweep_rows(P, X, rows, h4, 4.0, mu, **kw)
            bad = np.nonzero((cnt[:, :3] != oc[:, :3]).any(axis=1) |
                             ((cnt[:, 3] & 3) != (oc[:, 3] & 3)))[0]
            assert bad.size == 0, f"sweep {k + 1}: {bad.size} queries with other neighbour counts"
            e = float(np.abs(Xn - nxt).max())
            worst = max(worst, e)
            assert e <= 4 * eps * ext, f"sweep {k + 1}: off the reference map by {e:.3e}"
            X = Xn
    finally:
        plan.close()
    out = X
    print(f"cfg{cfg}: {its} sweeps shadow the reference map, worst step error "
          f"{worst / (eps * ext):.2f} ulp")

    r = orc.lop_project(P, X0, h4, 4.0, mu, its, store_f32=True, flags=True, **kw)
    tol = 1e-5 * bbox_diag(P)
    err = np.abs(out - r.points).max(axis=1)
    bad = err > tol
    # sensitivity of the reference's own trajectory to one ulp after sweep 1
    X1 = orc.lop_project(P, X0, h4, 4.0, mu, 1, store_f32=True, **kw).points
    rest = orc.lop_project(P, X1, h4, 4.0, mu, its - 1, store_f32=True, **kw).points
    sensitive = np.zeros(X0.shape[0], dtype=bool)
    own_beyond = 0
    perturbed = []
    for seed in (7, 8, 9):
        rng = np.random.default_rng(seed)
        away = np.where(rng.random(X1.shape) < 0.5, -np.inf, np.inf).astype(F32)
        X1j = np.nextafter(X1.astype(F32), away).astype(np.float64)
        rj = orc.lop_project(P, X1j, h4, 4.0, mu, its - 1, store_f32=True, **kw).points
        dj = np.abs(rj - rest).max(axis=1)
        sensitive |= dj > tol / 100
        own_beyond = max(own_beyond, int((dj > tol).sum()))
        perturbed.append(rj)
    event = ((gpu_ever & 6) != 0) | ((r.flags & (2 | 8)) != 0)
    near = np.zeros_like(bad)
    if bad.any() and event.any():
        from scipy.spatial import cKDTree
        t_ev = cKDTree(np.concatenate([r.points[event], out[event]]))
        d_ev = t_ev.query(np.concatenate([r.points[bad], out[bad]]))[0]
        nb = int(bad.sum())
        near[np.nonzero(bad)[0]] = np.minimum(d_ev[:nb], d_ev[nb:]) <= prm.kernel.support()
    unexplained = bad & ~sensitive & ~event & ~near
    print(f"cfg{cfg}: max err {err.max():.2e}, beyond tol {bad.sum()}/{len(err)} (sensitive "
          f"{int((bad & sensitive).sum())}, events {int((bad & (event | near)).sum())}, "
          f"unexplained {int(unexplained.sum())}); sensitive points {int(sensitive.sum())}; "
          f"oracle vs its 1-ulp-perturbed self beyond tol: up to {own_beyond}")
    assert unexplained.sum() == 0, np.nonzero(unexplained)[0][:10]
    assert bad.sum() <= 3 * own_beyond + 5
    if cfg in (3, 5):
        assert err.max() <= tol
    # and the projected sets are statistically the same surface sample: mean fit
    # distance and mean spacing within 1%, or within 1.5x the oracle's own spread
    # under the 1-ulp perturbations above (config 2: up to 0.84%)
    from scipy.spatial import cKDTree
    tP = cKDTree(P)
    fit = lambda X: tP.query(X)[0].mean()  # noqa: E731
    spacing = lambda X: cKDTree(X).query(X, k=2)[0][:, 1].mean()  # noqa: E731
    fit_gpu, fit_orc = fit(out), fit(r.points)
    sp_gpu, sp_orc = spacing(out), spacing(r.points)
    fit_spread = max([0.01 * fit_orc] + [1.5 * abs(fit(q) - fit(rest)) for q in perturbed])
    sp_spread = max([0.01 * sp_orc] + [1.5 * abs(spacing(q) - spacing(rest)) for q in perturbed])
    print(f"fit {fit_gpu:.5e} vs {fit_orc:.5e} (bound {fit_spread:.2e}); "
          f"spacing {sp_gpu:.5e} vs {sp_orc:.5e} (bound {sp_spread:.2e})")
    assert abs(fit_gpu - fit_orc) <= fit_spread
    assert abs(sp_gpu - sp_orc) <= sp_spread


# ----------------------------------------------------------------------------
# exact facilities
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_radius_queries_exact(pb, orc, prec):
    rng = np.random.default_rng(9)
    C = rng.uniform(-1, 1, (20000, 3))
    C[:100] = C[100:200]                                   # duplicated coordinates
    Q = np.concatenate([C[rng.choice(20000, 500)], rng.uniform(-3, 3, (100, 3))])  # far queries
    if prec == "fp32":
        C, Q = r32(C), r32(Q)
    for r in (0.02, 0.1, 0.35):
        off, idx = pb.radius_query_all(C, Q, r, precision=prec)
        o2, i2, _ = orc.radius_query_all(C, Q, r)
        assert np.array_equal(off, o2) and np.array_equal(idx, i2)


def test_radius_query_boundary_is_inclusive(pb):
    # proj/tests/test_spatial.cpp:21-30: d2 <= r*r exactly
    C = np.array([[0.0, 0, 0], [0.3, 0, 0], [np.nextafter(0.3, 1.0), 0, 0]])
    off, idx = pb.radius_query_all(C, np.zeros((1, 3)), 0.3)
    assert list(idx) == [0, 1]


def test_grid_sort_is_stable(pb):
    rng = np.random.default_rng(4)
    C = rng.uniform(-1, 1, (50000, 3))
    C[::7] = C[3]  # many equal keys
    keys, order = pb.grid_sort(C, 0.05)
    assert np.all(np.diff(keys.astype(np.int64)) >= 0)
    assert np.array_equal(np.sort(order), np.arange(len(C)))
    tie = keys[1:] == keys[:-1]
    assert np.all(order[1:][tie] > order[:-1][tie])


@pytest.mark.parametrize("prec,rtol", [("fp64", 1e-13), ("fp32", 2e-6)])
def test_density_weights(pb, orc, prec, rtol):
    P, _ = pb.generate_config(2, 0.01)
    P = r32(P)
    v = pb.density_weights(P, 0.075, 4.0, precision=prec)
    vo = orc.density_weights(P, 0.075, 4.0)
    assert np.abs(v / vo - 1).max() <= rtol


# ----------------------------------------------------------------------------
# semantics edge cases
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_coincident_and_duplicate_points(pb, orc, golden, prec):
    P = golden["lop_duplicates_P"]
    X0 = golden["lop_duplicates_X0"]
    if prec == "fp32":
        P, X0 = r32(P), r32(X0)
    h, cut, mu, it = golden["lop_duplicates_params"]
    prm = pb.LopParams(kernel=pb.KernelParams(h, cut), mu=mu, iterations=int(it))
    out, s = pb.lop_project(P, X0, prm, precision=prec)
    r = orc.lop_project(P, X0, h, cut, mu, int(it), store_f32=(prec == "fp32"))
    assert s.coincident_pairs == r.coincident_pairs > 0
    assert s.isolated_events == r.isolated_events
    assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_isolated_far_points(pb, orc, prec):
    rng = np.random.default_rng(5)
    P = r32(rng.uniform(-1, 1, (5000, 3)))
    X0 = r32(np.concatenate([P[:40], rng.uniform(5, 6, (5, 3))]))   # 5 isolated points
    prm = pb.LopParams(kernel=pb.KernelParams(0.05, 3.0), mu=0.0, iterations=3)
    out, s = pb.lop_project(P, X0, prm, precision=prec)
    r = orc.lop_project(P, X0, 0.05, 3.0, 0.0, 3, store_f32=(prec == "fp32"))
    assert s.isolated_indices == list(r.isolated_indices)
    assert {40, 41, 42, 43, 44} <= set(s.isolated_indices)
    assert s.isolated_events == r.isolated_events
    assert np.array_equal(out[40:], X0[40:])          # held in place (lop.cpp:70-73)
    assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)


def test_early_stop_on_convergence(pb, orc):
    # exact sphere samples, projected set lifted off the surface: the mu = 0
    # Weiszfeld iteration converges (oracle: 144 sweeps) below tol = 1e-6
    P = pb.generate_surface("sphere", 500, 3)
    rng = np.random.default_rng(6)
    X0 = P[rng.choice(500, 100, replace=False)] * 1.05
    prm = pb.LopParams(kernel=pb.KernelParams(0.5, 3.0), mu=0.0, iterations=400,
                       convergence_tol=1e-6)
    out, s = pb.lop_project(P, X0, prm, precision="fp64")
    r = orc.lop_project(P, X0, 0.5, 3.0, 0.0, 400, tol=1e-6)
    assert r.converged and s.converged
    assert abs(s.iterations_run - r.iterations_run) <= 1
    assert s.last_max_disp < 1e-6
    assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)


def test_determinism_and_plan_reset(pb):
    P, X0 = pb.generate_config(3, 0.01)
    prm, c = pb.config_params(3, h=0.2)
    a, sa = pb.lop_project(P, X0, prm, eta=c["eta"], precision="fp32")
    b, sb = pb.lop_project(P, X0, prm, eta=c["eta"], precision="fp32")
    assert np.array_equal(a, b) and sa.interactions_attr == sb.interactions_attr
    plan = pb.LopPlan(prm, eta=c["eta"], precision="fp32")
    plan.upload(P, X0)
    plan.run(5)
    plan.reset()
    plan.run(prm.iterations)
    c2, _ = plan.download()
    assert np.array_equal(a, c2)
    plan.close()


# ----------------------------------------------------------------------------
# layout / trimming edge cases of the fp32 kernels
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("offset", [(0.0, 0.0, 0.0), (512.0, -300.0, 800.0), (-4096.0, 17.0, 0.5)])
def test_fp32_neighbours_exact_far_from_origin(pb, orc, offset):
    """Row trimming runs in fp32 with a slack of 32 ulps of the coordinate scale;
    far from the origin fp32 rounding is large relative to the support, and the
    neighbour sets must still be the reference's (identical counts)."""
    P, X0 = pb.generate_config(3, 0.004)
    off = np.array(offset)
    P, X0 = r32(P + off), r32(X0 + off)
    prm, c = pb.config_params(3, h=0.2)
    prm.iterations = 1
    out, s = pb.lop_project(P, X0, prm, eta=c["eta"], precision="fp32")
    r = orc.lop_project(P, X0, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu, 1,
                        eta=orc.ETA_NEG_LINEAR, store_f32=True)
    assert (s.interactions_attr, s.interactions_rep) == (r.interactions_attr, r.interactions_rep)
    assert np.abs(out - r.points).max() <= 8 * np.finfo(F32).eps * np.abs(P).max()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_plan_with_tiny_projected_sets(pb, orc, prec):
    """m = 0, 1, 2 through the plan API (empty work lists, one-point groups)."""
    P, _ = pb.generate_config(3, 0.002)
    prm, c = pb.config_params(3, h=0.2)
    prm.iterations = 3
    for m in (0, 1, 2):
        X0 = P[:m] + 1e-3
        plan = pb.LopPlan(prm, eta=c["eta"], precision=prec)
        plan.upload(P, X0)
        plan.run(3)
        out, s = plan.download()
        plan.close()
        assert out.shape == (m, 3)
        if m:
            r = orc.lop_project(r32(P) if prec == "fp32" else P, r32(X0) if prec == "fp32" else X0,
                                prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu, 3,
                                eta=orc.ETA_NEG_LINEAR, store_f32=(prec == "fp32"))
            assert s.interactions_attr == r.interactions_attr
            assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)


def test_mu0_skips_projected_grid_but_matches(pb, orc):
    """mu = 0: one fused pass, no projected-set grid; same result as the oracle."""
    P, X0, prm, c = scaled_case(pb, 5, 0.001, 0.3)
    prm.mu = 0.0
    prm.iterations = 2
    out, s = pb.lop_project(P, X0, prm, eta=c["eta"], precision="fp32")
    r = orc.lop_project(P, X0, prm.kernel.h, prm.kernel.cutoff_multiple, 0.0, 2,
                        eta=orc.ETA_INV_CUBE, store_f32=True)
    assert s.interactions_attr == r.interactions_attr and s.interactions_rep == 0
    assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)


@pytest.mark.parametrize("shape", ["line", "plane_grid", "clustered"])
def test_fp32_degenerate_geometry_exact_neighbours(pb, orc, shape):
    """Degenerate clouds through the fp32 plan (Hilbert order, bisected groups,
    zero-extent axes, ties in every sort key): one sweep has the oracle's
    neighbour sets exactly and agrees to fp32 rounding."""
    rng = np.random.default_rng(41)
    if shape == "line":
        P = np.zeros((4000, 3))
        P[:, 0] = rng.uniform(-1, 1, 4000)
    elif shape == "plane_grid":
        g = np.arange(60) * 0.02
        P = np.stack(np.meshgrid(g, g, [0.5]), -1).reshape(-1, 3)
    else:  # a few tight clusters with many coincident points
        c = rng.uniform(-1, 1, (6, 3))
        P = np.repeat(c, 500, axis=0) + rng.normal(scale=0.01, size=(3000, 3))
        P[::7] = P[1::7]
    P = r32(P)
    X0 = P[rng.choice(P.shape[0], P.shape[0] // 10, replace=False)]
    prm, c = pb.config_params(3, h=0.06)
    prm.iterations = 1
    out, s = pb.lop_project(P, X0, prm, eta=c["eta"], precision="fp32")
    r = orc.lop_project(P, X0, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu, 1,
                        eta=orc.ETA_NEG_LINEAR, store_f32=True)
    assert (s.interactions_attr, s.interactions_rep) == (r.interactions_attr, r.interactions_rep)
    assert (s.isolated_events, s.coincident_pairs) == (r.isolated_events, r.coincident_pairs)
    assert np.abs(out - r.points).max() <= 4 * np.finfo(F32).eps * max(np.abs(P).max(), 1.0)


@pytest.mark.parametrize("wlop", [False, True])
def test_deferred_queries_match_oracle(pb, orc, wlop):
    """Projected points sitting exactly on a lonely data point stay anchored
    there (lop.cpp:67-69); from sweep 2 on the fp32 kernel meets their exact
    zero distance and defers them to the exact kernel (a block per query).
    Their result, and everyone else's, must match the oracle."""
    rng = np.random.default_rng(11)
    # a well-conditioned surface sample (~350 neighbours per point: no iterate
    # lands on a data sample, see test_fp32_full_trajectory) ...
    dense = rng.uniform(-1, 1, (20000, 3)) * np.array([1.0, 1.0, 0.01])
    g = np.arange(4) * 0.2                      # 64 points 0.2 > s apart, off the cloud
    lonely = 1.3 + np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    P = r32(np.concatenate([dense, lonely]))
    X0 = r32(np.concatenate([P[:300], P[20000:]]))   # ... and the lonely points
    prm = pb.LopParams(kernel=pb.KernelParams(0.05, 3.0), mu=0.4, iterations=4)
    eta = "neg_linear" if wlop else "inv_cube"
    out, s = pb.lop_project(P, X0, prm, eta=eta, density_weights=wlop, precision="fp32")
    r = orc.lop_project(P, X0, 0.05, 3.0, 0.4, 4, store_f32=True, wlop=wlop,
                        eta=orc.ETA_NEG_LINEAR if wlop else orc.ETA_INV_CUBE)
    assert s.careful_points >= 64 * 3          # the lonely points, sweeps 2..4
    assert (s.interactions_attr, s.interactions_rep) == (r.interactions_attr, r.interactions_rep)
    assert (s.isolated_events, s.coincident_pairs) == (r.isolated_events, r.coincident_pairs)
    assert np.array_equal(out[300:], X0[300:])  # anchored on themselves
    assert np.abs(out - r.points).max() <= 1e-5 * bbox_diag(P)


@pytest.mark.parametrize("cfg,scale,h,prec", [(3, 0.01, 0.2, "fp32"), (2, 0.02, 0.3, "fp32"),
                                              (1, 1.0, None, "fp64")])
def test_cuda_graph_replay_is_bit_identical(pb, cfg, scale, h, prec):
    """Sweeps 2.. replayed as captured CUDA graphs of 8 sweeps give exactly the
    positions and summary of enqueuing every launch (deterministic kernels, same
    launch order).  The first run with graphs on enqueues every launch and
    captures the period at its end (off the critical path); the next run
    replays it (graph launches counted)."""
    P, X0 = pb.generate_config(cfg, scale)
    if prec == "fp32":
        P, X0 = r32(P), r32(X0)
    prm, c = pb.config_params(cfg, h=h)
    prm.iterations = 21
    prm.convergence_tol = 1e-30
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision=prec)
    try:
        plan.upload(P, X0)
        res = {}
        for on in (False, True, True):
            plan.set_graphs(on)
            plan.reset()
            g0 = plan.graph_launches()
            plan.run(21)
            out, s = plan.download()
            res.setdefault(on, []).append((out, s, plan.graph_launches() - g0))
        (o0, s0, g_off), = res[False]
        assert [g for _, _, g in res[True]] == [0, 2]  # then sweeps 2-9 and 10-17 replayed
        for out, s, g in res[True]:
            assert np.array_equal(out, o0)
            assert (s.iterations_run, s.interactions_attr, s.interactions_rep, s.isolated_events,
                    s.coincident_pairs, s.careful_points) == \
                   (s0.iterations_run, s0.interactions_attr, s0.interactions_rep,
                    s0.isolated_events, s0.coincident_pairs, s0.careful_points)
        assert g_off == 0
    finally:
        plan.close()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_positions_outside_the_upload_box(pb, orc, prec):
    """Projected points may leave the box the grids were built over (repulsion
    pushes boundary points outward; an isolated point holds its position): out-
    of-range cells clamp into the boundary cells, which are unbounded outward,
    so no neighbour is lost (SURVEY §8(a') item 7).  The plan restarts from
    positions placed outside the upload-time box — far away (isolated), and
    just outside, within one support of the data — and one sweep must equal the
    reference map per query (counts exact, positions within rounding)."""
    P, X0 = pb.generate_config(3, 0.01)
    if prec == "fp32":
        P, X0 = r32(P), r32(X0)
    prm, c = pb.config_params(3, h=0.2)
    s = prm.kernel.support()
    lo, hi = np.minimum(P.min(0), X0.min(0)), np.maximum(P.max(0), X0.max(0))
    X = X0.copy()
    X[:40] += np.array([3.0, 0.0, 0.0])                       # far beyond +x: isolated
    X[40:80] += np.array([0.0, -2.5, 0.7])                    # far beyond -y, +z
    edge = np.argsort(P[:, 0])[-40:]                          # data points at the +x edge
    X[80:120] = P[edge] + np.array([0.6 * s, 0.0, 0.25 * s])  # outside the box, data within s
    edge = np.argsort(P[:, 1])[:40]
    X[120:160] = P[edge] - np.array([0.0, 0.45 * s, 0.0])
    if prec == "fp32":
        X = r32(X)
    assert ((X[:160] < lo) | (X[:160] > hi)).any(axis=1).all()
    plan = pb.LopPlan(prm, eta=c["eta"], precision=prec)
    try:
        plan.upload(P, X0)
        plan.set_positions(X)
        plan.record_counts(True)
        plan.run(1)
        Xn, _ = plan.download()
        cnt, _ = plan.query_counts()
    finally:
        plan.close()
    eta = orc.ETA_NEG_LINEAR
    rows = np.arange(X.shape[0], dtype=np.uint32)
    nxt, oc = orc.lop_sweep_rows(P, X, rows, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu,
                                 eta=eta)
    assert np.array_equal(cnt[:, :3], oc[:, :3])
    assert np.array_equal(cnt[:, 3] & 3, oc[:, 3] & 3)
    assert (oc[:80, 3] & 1).all() and (oc[80:160, 0] > 0).all()  # isolated far; edge ones attracted
    tol = 4 * np.finfo(np.float32).eps * np.abs(X).max() if prec == "fp32" else 1e-12
    assert np.abs(Xn - nxt).max() <= tol
