"""Multi-rank host logic on CPU (gloo, world_size 2).

The GPU plan shards X by contiguous ranges of its initial grid order
(pcs_shard_layout, paper_2401_03365_b200/csrc/shard.cpp): each rank updates its
own internal slots, then one in-place all-gather of `chunk` points per rank
rebuilds X^{k+1} on every rank, and the max displacement is all-reduced (MAX).
Here the same layout function drives a 2-process emulation in which each rank
computes only its own shard of each Jacobi sweep (oracle arithmetic), exchanges
shards with torch.distributed (gloo) and must reproduce the single-process
sweeps bit-for-bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sweeps, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import oracle as O
    import paper_2401_03365_b200 as pb

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(11)
    P = rng.uniform(-1, 1, (3000, 3))
    P[:, 2] *= 0.1
    X0 = P[rng.choice(3000, 301, replace=False)]
    h, cut, mu = 0.05, 4.0, 0.4
    # the "grid order" of X0: stable sort by a coarse cell key (any permutation is valid)
    cell = np.floor((X0 + 1.0) / 0.2).astype(np.int64)
    key = cell[:, 0] + 16 * (cell[:, 1] + 16 * cell[:, 2])
    order = np.argsort(key, kind="stable")
    chunk, counts, ooi, ioo = pb.shard_layout(order, world)
    lo = rank * chunk
    own_slots = np.arange(lo, lo + counts[rank])
    own_orig = ooi[own_slots]

    X = X0.copy()
    ever_iso = np.zeros(len(X0), dtype=np.uint8)
    ok = True
    for k in range(sweeps):
        # this rank's shard of the Jacobi sweep (lop.cpp:41-100): rows own_orig only
        nxt, iso, co, _ = O.lop_sweep(P, X, h, cut, mu, eta=O.ETA_NEG_LINEAR)
        send = np.full((chunk, 3), np.nan)
        send[: counts[rank]] = nxt[own_orig]
        disp = np.linalg.norm(nxt[own_orig] - X[own_orig], axis=1).max(initial=0.0)
        # in-place all-gather of the internal layout, then the max-displacement all-reduce
        parts = [torch.empty((chunk, 3), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(send))
        internal = torch.cat(parts).numpy()
        md = torch.tensor([disp], dtype=torch.float64)
        dist.all_reduce(md, op=dist.ReduceOp.MAX)
        iso_own = np.zeros(len(X0), dtype=np.uint8)
        iso_own[own_orig] = iso[own_orig]
        iso_t = torch.from_numpy(iso_own.astype(np.int32))
        dist.all_reduce(iso_t, op=dist.ReduceOp.MAX)
        ever_iso |= iso_t.numpy().astype(np.uint8)
        Xn = internal[ioo]                       # internal -> original order
        # single-process reference sweep
        full, iso_full, _, md_full = O.lop_sweep(P, X, h, cut, mu, eta=O.ETA_NEG_LINEAR)
        ok &= bool(np.array_equal(Xn, full))
        ok &= bool(md.item() == md_full)
        ok &= bool(np.array_equal(iso_t.numpy().astype(np.uint8), iso_full))
        X = Xn
    out_q.put((rank, ok, int(chunk), [int(c) for c in counts]))
    dist.destroy_process_group()


def test_two_rank_sharded_sweeps_match_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, t0 = [], time.time()
    while len(res) < world and time.time() - t0 < 300:
        try:
            res.append(q.get(timeout=1))
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res) == world
    for rank, ok, chunk, counts in res:
        assert ok, f"rank {rank} diverged from the single-process sweep"
        assert chunk == 151 and sum(counts) == 301


def test_shard_layout_properties(pb):
    rng = np.random.default_rng(3)
    for m, world in [(0, 1), (1, 4), (10, 3), (1000, 8), (1001, 7)]:
        order = rng.permutation(m).astype(np.uint32)
        chunk, counts, ooi, ioo = pb.shard_layout(order, world)
        assert counts.sum() == m and chunk * world >= m and counts.max() <= chunk
        valid = ooi != 0xFFFFFFFF
        assert valid.sum() == m
        assert np.array_equal(np.sort(ooi[valid]), np.arange(m))
        if m:
            assert np.array_equal(ooi[ioo], np.arange(m))
            # shards are contiguous ranges of the sorted order
            r = ioo[order] // chunk
            assert np.all(np.diff(r.astype(np.int64)) >= 0)
    with pytest.raises(pb.InvalidParam):
        pb.shard_layout(np.array([5, 1], dtype=np.uint32), 2)   # not a permutation of 0..m-1


def test_weighted_shard_layout_balances_work(pb):
    """Cuts at equal cumulative work: contiguous ranges of the sorted
    order, every rank's work within one point's weight of the ideal share."""
    rng = np.random.default_rng(9)
    for m, world in [(1, 4), (10, 3), (5000, 8), (4001, 7)]:
        order = rng.permutation(m).astype(np.uint32)
        # density rising 50x along the sorted order, like config 4's pole
        w = np.exp(3.9 * np.linspace(-1, 1, m)).astype(np.float32)[np.argsort(order)]
        chunk, counts, ooi, ioo = pb.shard_layout(order, world, weights=w)
        assert counts.sum() == m and counts.max() == chunk
        valid = ooi != 0xFFFFFFFF
        assert np.array_equal(np.sort(ooi[valid]), np.arange(m))
        assert np.array_equal(ooi[ioo], np.arange(m))
        r = ioo[order] // chunk
        assert np.all(np.diff(r.astype(np.int64)) >= 0)
        if m >= world:
            share = np.array([w[ooi[k * chunk:k * chunk + counts[k]]].sum() for k in range(world)])
            assert np.abs(share - w.sum() / world).max() <= w.max() + 1e-3 * w.sum()
        if m > 100:  # unequal counts: the dense end gets fewer points per rank
            assert counts[0] > counts[-1]
    # unit weights = near-equal counts
    order = rng.permutation(1000).astype(np.uint32)
    _, counts, _, _ = pb.shard_layout(order, 8, weights=np.ones(1000, np.float32))
    assert counts.max() - counts.min() <= 1


def test_weighted_layout_evens_config4_work(pb):
    """Config 4 (density ~ e^{3.9z}): with equal-count shards the rank holding the
    dense pole does several times the mean work; cutting at the density proxy the
    plans use (data points in the 3x3x3 cells of side s/4 around each point)
    brings the max/mean work ratio near 1.  Work = true neighbour counts."""
    from scipy.spatial import cKDTree
    P, X0 = pb.generate_config(4, 0.01)
    s = 0.03
    work = np.array([len(l) for l in cKDTree(P).query_ball_point(X0, s)], dtype=np.float64)
    cs = s / 4
    lo = np.minimum(P.min(0), X0.min(0)) - cs
    cP = np.floor((P - lo) / cs).astype(np.int64)
    cX = np.floor((X0 - lo) / cs).astype(np.int64)
    from collections import Counter
    cnt = Counter(map(tuple, cP))
    proxy = np.array([1 + sum(cnt.get((x + a, y + b, z + c), 0) for a in (-1, 0, 1)
                              for b in (-1, 0, 1) for c in (-1, 0, 1)) for x, y, z in cX],
                     dtype=np.float32)
    g = (cX[:, 2] * 10000 + cX[:, 1]) * 10000 + cX[:, 0]   # cell order (x fastest)
    order = np.argsort(g, kind="stable").astype(np.uint32)
    world = 8

    def imbalance(weights):
        chunk, counts, ooi, _ = pb.shard_layout(order, world, weights=weights)
        per = [work[ooi[k * chunk:k * chunk + counts[k]]].sum() for k in range(world)]
        return max(per) / (sum(per) / world)

    equal, weighted = imbalance(None), imbalance(proxy)
    assert equal > 1.5
    assert weighted < 1.25 and weighted < equal
