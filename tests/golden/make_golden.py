"""Generates tests/golden/reference_cases.npz from the UNMODIFIED reference.

Run in the container that has /root/reference (the reference is compiled from
its own sources into oracle/_ref by `make -C oracle ref`):

    python tests/golden/make_golden.py

Every array in the fixture is an output of the reference's own functions
(pcs::generate_surface, pcs::add_noise, pcs::SpatialIndex::radius_query,
pcs::lop_project) on seeded inputs; the inputs are stored beside them.  The
fixture pins the oracle (oracle/lop_oracle.c) bit-for-bit and the B200 path
within tolerance, on boxes where /root/reference does not exist.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def fy_subset(P, m, seed):
    rng = np.random.default_rng(seed)
    return P[np.sort(rng.choice(P.shape[0], m, replace=False))]


def main() -> None:
    O.build(reference=True)
    assert O.ref_available(), "oracle/_ref not built (needs /root/reference)"
    out = {}
    # generators (proj/src/bench.cpp:40-87) and noise (proj/src/noise.cpp:9-27)
    for kind in range(4):
        out[f"surface_{kind}"] = O.ref_generate_surface(kind, 100, 7)
    base = O.ref_generate_surface(1, 50, 3)
    out["noise_in"] = base
    out["noise_out"] = O.ref_add_noise(base, 0.1, 9)
    out["noise_kat"] = O.ref_add_noise(np.zeros((1, 3)), 1.0, 1)  # test_noise.cpp:64-72

    # radius queries (proj/src/spatial.cpp:82-111)
    rng = np.random.default_rng(5)
    C = rng.uniform(-1, 1, (400, 3))
    C[10] = C[11]  # duplicate coordinates (test_spatial.cpp:113-124)
    Q = np.concatenate([rng.uniform(-1.2, 1.2, (38, 3)), C[10:12]])
    off, idx, dist = O.ref_radius_query_all(C, Q, 0.3)
    out.update(rq_cloud=C, rq_queries=Q, rq_r=np.array(0.3), rq_offsets=off, rq_idx=idx,
               rq_dist=dist)

    # lop_project (proj/src/lop.cpp:10-127), seeded cases
    cases = {}
    D = O.ref_add_noise(O.ref_generate_surface(0, 2000, 11), 0.05, 55)
    cases["plane"] = (D, D[::10][:200], 0.3, 3.0, 0.4, 30)
    cases["single"] = (np.array([[0.3, -0.2, 0.8]]), np.array([[0.5, 0.1, 0.6]]), 1.0, 3.0, 0.0, 30)
    cases["pair"] = (np.array([[-1.0, 0, 0], [1.0, 0, 0]]), np.array([[0, 0.5, 0.0]]), 10.0, 3.0,
                     0.0, 60)
    cases["isolated"] = (np.array([[0.0, 0, 0]]), np.array([[5.0, 0, 0]]), 0.1, 3.0, 0.0, 30)
    cases["coincident"] = (np.array([[1.0, 2, 3]]), np.array([[1.0, 2, 3]]), 0.5, 3.0, 0.0, 30)
    R = rng.uniform(-1, 1, (200, 3))
    cases["random"] = (R, rng.uniform(-0.8, 0.8, (20, 3)), 0.25, 3.0, 0.3, 10)
    S = O.ref_add_noise(O.ref_generate_surface(1, 2000, 0), 0.01, 1)
    cases["sphere"] = (S, fy_subset(S, 200, 2), 0.3 / 4, 4.0, 0.45, 5)
    Dup = np.concatenate([S[:300], S[:50]])            # duplicated data samples
    X0d = np.concatenate([S[:20], S[:5], S[100:110]])  # coincident projected points
    cases["duplicates"] = (Dup, X0d, 0.3 / 4, 4.0, 0.45, 4)
    for name, (P, X0, h, cut, mu, it) in cases.items():
        r = O.ref_lop_project(P, X0, h, cut, mu, it)
        out[f"lop_{name}_P"] = P
        out[f"lop_{name}_X0"] = X0
        out[f"lop_{name}_params"] = np.array([h, cut, mu, it], dtype=np.float64)
        out[f"lop_{name}_out"] = r.points
        out[f"lop_{name}_summary"] = np.array([r.iterations_run, int(r.converged),
                                               r.isolated_events, r.coincident_pairs],
                                              dtype=np.int64)
        out[f"lop_{name}_isolated"] = np.asarray(r.isolated_indices, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "reference_cases.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_cases.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
