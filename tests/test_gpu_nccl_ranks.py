"""Sharded plans over NCCL with one process per GPU (GPU, needs >= 2 devices).

The multi-GPU design of SURVEY.md §8(e): every rank holds P and X0, owns a
contiguous, work-weighted range of X0's grid order, updates it, and one
in-place NCCL all-gather per sweep (plus a max all-reduce of the displacement)
rebuilds X on every rank.  Two ranks on two GPUs must reproduce the
single-GPU run: identical interaction / density / isolation counts and sweep
counts, positions equal up to fp32 summation order.  Skipped on a one-GPU box
(the loopback and 1-rank NCCL tests of test_gpu_sharded.py cover the same plan
code there).
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _rank(rank, world, uid, cfg, scale, out_q):
    sys.path.insert(0, ROOT)
    import paper_2401_03365_b200 as pb
    P, X0 = pb.generate_config(cfg, scale)
    prm, c = pb.config_params(cfg)
    prm.iterations = 5
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32", device=rank)
    plan.set_comm(uid, world, rank)
    plan.upload(P, X0)
    plan.run(prm.iterations)
    X, s = plan.download()
    plan.close()
    out_q.put((rank, X, (s.iterations_run, s.interactions_attr, s.interactions_rep,
                         s.density_pairs, tuple(s.isolated_indices))))


@pytest.mark.skipif(_ngpus() < 2, reason="needs two GPUs (one process per GPU)")
@pytest.mark.parametrize("cfg,scale", [(3, 0.01), (4, 0.02)])
def test_two_gpu_nccl_ranks_match_single_gpu(pb, cfg, scale):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = pb.LopPlan.nccl_unique_id()
    procs = [ctx.Process(target=_rank, args=(r, 2, uid, cfg, scale, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    P, X0 = pb.generate_config(cfg, scale)
    prm, c = pb.config_params(cfg)
    prm.iterations = 5
    ref, s = pb.lop_project(P, X0, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32",
                            device=0)
    want = (s.iterations_run, s.interactions_attr, s.interactions_rep, s.density_pairs,
            tuple(s.isolated_indices))
    diag = float(np.linalg.norm(P.max(0) - P.min(0)))
    for rank, X, summary in res:
        assert summary == want, (rank, summary, want)
        assert np.abs(X - ref).max() <= 1e-6 * diag
