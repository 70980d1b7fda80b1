"""Oracle parity of the fused fp32 path at the BASELINE configurations' full
sizes and h (GPU).

The function whose outputs must match is the per-point body of the reference
sweep, /root/reference/proj/src/lop.cpp:41-100, on the neighbour sets of
SpatialIndex::radius_query (proj/src/spatial.cpp:82-111).  At full size the
oracle cannot afford every query, so it evaluates a seeded subset of rows of
the same sweep (oracle orc_lop_sweep_rows: all of P and all of X^k are the
candidates) and the B200 plan reports, per query, what its fused kernel (or
the exact kernel, for deferred queries) actually counted
(pcs_lop_plan_query_counts).  Per row:

* attraction interactions (0 < d <= s), repulsion interactions, coincident
  pairs and the isolated / anchored flags are EXACT (the neighbour sets are the
  reference's: a compensating per-query error cannot hide in a total);
* the new position is within 4 fp32 ulps of the coordinate scale.

Each configuration is checked for the first sweep (from X0) and for one sweep
from the GPU's own state after k sweeps (k = the configuration's iteration
count minus one), and the per-query counts of every row also sum, over ALL
queries, to the run's interaction totals.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

F32 = np.float32
EPS32 = float(np.finfo(F32).eps)
ROWS = 20000

# (config, h = support or None for the BASELINE value, k = sweeps before the second check)
FULL = [(3, None, 14), (5, 0.01, 9), (2, None, 29), (4, None, 19)]


def r32(a):
    return np.asarray(a, dtype=F32).astype(np.float64)


def check_sweep(orc, P, X, Xn, counts, rows, prm, c, label):
    eta = orc.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else orc.ETA_INV_CUBE
    nxt, oc = orc.lop_sweep_rows(P, X, rows, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu,
                                 eta=eta, wlop=c["wlop"])
    g = counts[rows]
    assert (g[:, 0] >= 0).all(), f"{label}: rows without a record"
    bad = np.nonzero((g[:, :3] != oc[:, :3]).any(axis=1) | ((g[:, 3] & 3) != (oc[:, 3] & 3)))[0]
    assert bad.size == 0, (f"{label}: {bad.size} rows differ, e.g. row {rows[bad[0]]}: "
                           f"B200 {g[bad[0]]} oracle {oc[bad[0]]}")
    ext = float(np.abs(P).max())
    err = np.abs(Xn[rows] - nxt).max(axis=1)
    worst = int(np.argmax(err))
    print(f"{label}: {rows.size} rows, attraction {int(oc[:, 0].sum())} repulsion "
          f"{int(oc[:, 1].sum())} interactions identical; max position error "
          f"{err.max():.3e} ({err.max() / (EPS32 * ext):.2f} ulp of {ext:.3f}); "
          f"deferred rows {int(((g[:, 3] & 4) != 0).sum())}")
    assert err.max() <= 4 * EPS32 * ext, f"{label}: row {rows[worst]} off by {err[worst]:.3e}"


@pytest.mark.parametrize("cfg,h,k", FULL)
def test_full_size_per_query_parity(pb, orc, cfg, h, k):
    P, X0 = pb.generate_config(cfg)
    P, X0 = r32(P), r32(X0)
    prm, c = pb.config_params(cfg, h=h)
    rng = np.random.default_rng(1000 + cfg)
    rows = np.sort(rng.choice(X0.shape[0], ROWS, replace=False)).astype(np.uint32)
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32", device=0)
    try:
        plan.upload(P, X0)
        plan.record_counts(True)
        # sweep 1 from X0
        plan.run(1)
        X1, s1 = plan.download()
        cnt1, _ = plan.query_counts()
        assert cnt1[:, 0].sum() == s1.interactions_attr
        assert cnt1[:, 1].sum() == s1.interactions_rep
        check_sweep(orc, P, X0, X1, cnt1, rows, prm, c, f"config {cfg} sweep 1")
        # one sweep from the GPU's own state after k sweeps
        if k > 1:
            plan.run(k - 1)
        Xk, sk = plan.download()
        plan.run(1)
        Xk1, sk1 = plan.download()
        cnt, _ = plan.query_counts()
        assert sk1.iterations_run == k + 1, "converged early: nothing left to check"
        assert cnt[:, 0].sum() == sk1.interactions_attr - sk.interactions_attr
        assert cnt[:, 1].sum() == sk1.interactions_rep - sk.interactions_rep
        check_sweep(orc, P, Xk, Xk1, cnt, rows, prm, c, f"config {cfg} sweep {k + 1}")
    finally:
        plan.close()
