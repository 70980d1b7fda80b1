"""Sharded (multi-rank) plan path on one B200 through loopback groups.

The plan code that runs per rank under NCCL (ownership layout, Morton query
list with owned queries first, partial Jacobi updates, in-place all-gather of
X, max-reduce of the displacement, counter/isolation reduction at download —
SURVEY.md §8e) runs here with R ranks as R threads of one
process; only the transport differs (device-to-device copies instead of NCCL).
Results must match the single-rank run: identical interaction/isolation
counts and sweep counts, positions equal up to fp32 summation order.
"""
import threading

import numpy as np
import pytest

import paper_2401_03365_b200 as pb

pytestmark = pytest.mark.gpu


def _sharded(P, X0, prm, nranks, **kw):
    group = pb.LoopbackGroup(nranks)
    plans = [pb.LopPlan(prm, **kw) for _ in range(nranks)]
    for r, p in enumerate(plans):
        p.set_loopback(group, r)
    out = [None] * nranks
    err = []

    def work(r):
        try:
            plans[r].upload(P, X0)
            plans[r].run(prm.iterations)
            out[r] = plans[r].download()
        except Exception as e:  # surfaced below
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    for p in plans:
        p.close()
    return out


def _single(P, X0, prm, **kw):
    plan = pb.LopPlan(prm, **kw)
    plan.upload(P, X0)
    plan.run(prm.iterations)
    res = plan.download()
    plan.close()
    return res


@pytest.mark.parametrize("cfg,scale,nranks", [(3, 0.01, 2), (5, 0.002, 3), (2, 0.05, 2), (4, 0.02, 4)])
def test_loopback_ranks_match_single_gpu(cfg, scale, nranks):
    P, X0 = pb.generate_config(cfg, scale)
    prm, c = pb.config_params(cfg)
    prm.iterations = 4
    kw = dict(eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    ref, sref = _single(P, X0, prm, **kw)
    diag = float(np.linalg.norm(P.max(0) - P.min(0)))
    outs = _sharded(P, X0, prm, nranks, **kw)
    for X, s in outs:  # every rank returns the full projected set and job totals
        assert s.iterations_run == sref.iterations_run
        assert s.interactions_attr == sref.interactions_attr
        assert s.interactions_rep == sref.interactions_rep
        assert s.isolated_events == sref.isolated_events
        assert s.isolated_indices == sref.isolated_indices
        assert s.careful_points == sref.careful_points
        if c["wlop"]:
            assert s.density_pairs == sref.density_pairs
        # identical neighbour sets (counts above); positions differ only by the fp32
        # summation order, which follows the query grouping (the ranks' query
        # lists differ from the single GPU's) — bounded by the parity tolerance
        err = np.abs(X - ref).max()
        assert err <= 1e-5 * diag, (cfg, nranks, err / diag)
    # all ranks agree bit-for-bit with each other (same all-gathered state)
    for X, _ in outs[1:]:
        assert np.array_equal(X, outs[0][0])


def test_loopback_early_stop_consistent_fp64():
    """fp64 (exact kernel) sharded path; convergence is decided on the all-reduced
    displacement, so every rank stops at the same sweep as one GPU does."""
    P = pb.generate_surface("sphere", 500, 3)
    rng = np.random.default_rng(6)
    X0 = P[rng.choice(500, 100, replace=False)] * 1.05
    prm = pb.LopParams(kernel=pb.KernelParams(0.5, 3.0), mu=0.0, iterations=400,
                       convergence_tol=1e-6)
    kw = dict(eta="inv_cube", precision="fp64")
    ref, sref = _single(P, X0, prm, **kw)
    outs = _sharded(P, X0, prm, 2, **kw)
    assert sref.converged
    for X, s in outs:
        assert s.converged and s.iterations_run == sref.iterations_run
        assert s.interactions_attr == sref.interactions_attr
        assert np.abs(X - ref).max() <= 1e-12 * float(np.linalg.norm(P.max(0) - P.min(0)))


def test_loopback_fp64_lop_config1():
    """Config 1 (the reference's CPU-runnable case, fp64) on 3 ranks == 1 rank."""
    P, X0 = pb.generate_config(1, 0.25)
    prm, c = pb.config_params(1)
    prm.iterations = 5
    kw = dict(eta=c["eta"], precision="fp64")
    ref, sref = _single(P, X0, prm, **kw)
    for X, s in _sharded(P, X0, prm, 3, **kw):
        assert s.interactions_attr == sref.interactions_attr
        assert s.interactions_rep == sref.interactions_rep
        assert s.coincident_pairs == sref.coincident_pairs
        assert s.isolated_indices == sref.isolated_indices
        assert np.abs(X - ref).max() <= 1e-12 * float(np.linalg.norm(P.max(0) - P.min(0)))


def test_nccl_single_rank_clique_matches_plain_run():
    """A 1-rank NCCL clique runs the sharded plan path with real NCCL calls
    (dlopen'ed libnccl, in-place all-gather, uint64 max/sum and uint8 max
    all-reduces) on one GPU.  The sharded layout renumbers points (ties inside a
    grid cell sort by that number), so only the fp32 summation order differs."""
    P, X0 = pb.generate_config(4, 0.01)
    prm, c = pb.config_params(4)
    prm.iterations = 3
    kw = dict(eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    ref, sref = _single(P, X0, prm, **kw)
    plan = pb.LopPlan(prm, **kw)
    plan.set_comm(pb.LopPlan.nccl_unique_id(), 1, 0)
    plan.upload(P, X0)
    plan.run(prm.iterations)
    X, s = plan.download()
    plan.close()
    assert np.abs(X - ref).max() <= 1e-6 * float(np.linalg.norm(P.max(0) - P.min(0)))
    assert s.interactions_attr == sref.interactions_attr
    assert s.interactions_rep == sref.interactions_rep
    assert s.density_pairs == sref.density_pairs
