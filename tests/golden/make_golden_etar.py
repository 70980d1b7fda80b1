"""Generates tests/golden/reference_etar.npz: LOP cases with eta(r) = -r, run
by the reference's own lop.cpp (oracle/_ref/libpcs_ref_etar.so — the
unmodified reference objects with lop.cpp's |eta'| call bound to |eta'| = 1 by
`-Wl,--wrap`, see oracle/ref_etar_wrap.cpp).

    python tests/golden/make_golden_etar.py

Pins the eta = -r variant (benchmark configs 2-4) of the oracle bit-for-bit and
of the B200 path within tolerance on boxes without /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def main() -> None:
    O.build(reference=True)
    eta = O.ETA_NEG_LINEAR
    out = {}
    cases = {}
    rng = np.random.default_rng(21)
    # the height field of config 3 (reduced), fp32-rounded as the fp32 path sees it
    P3, X3 = O.generate_config(3, 0.002)
    P3 = P3.astype(np.float32).astype(np.float64)
    X3 = X3.astype(np.float32).astype(np.float64)
    cases["height"] = (P3, X3, 0.2 / 4, 4.0, 0.4, 6)
    S = O.ref_add_noise(O.ref_generate_surface(1, 3000, 0), 0.01, 1)
    cases["sphere"] = (S, S[rng.choice(3000, 300, replace=False)], 0.3 / 4, 4.0, 0.45, 8)
    Dup = np.concatenate([S[:400], S[:60]])             # duplicated data samples
    X0d = np.concatenate([S[:30], S[:6], S[200:215]])   # coincident projected points
    cases["duplicates"] = (Dup, X0d, 0.3 / 4, 4.0, 0.45, 4)
    R = rng.uniform(-1, 1, (300, 3))
    far = rng.uniform(4, 5, (4, 3))                     # isolated queries
    cases["random_isolated"] = (R, np.concatenate([rng.uniform(-0.8, 0.8, (25, 3)), far]),
                                0.25, 3.0, 0.3, 10)
    for name, (P, X0, h, cut, mu, it) in cases.items():
        r = O.ref_lop_project(P, X0, h, cut, mu, it, eta=eta)
        out[f"lop_{name}_P"] = P
        out[f"lop_{name}_X0"] = X0
        out[f"lop_{name}_params"] = np.array([h, cut, mu, it], dtype=np.float64)
        out[f"lop_{name}_out"] = r.points
        out[f"lop_{name}_summary"] = np.array([r.iterations_run, int(r.converged),
                                               r.isolated_events, r.coincident_pairs],
                                              dtype=np.int64)
        out[f"lop_{name}_isolated"] = np.asarray(r.isolated_indices, dtype=np.int64)
    path = os.path.join(HERE, "reference_etar.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays")


if __name__ == "__main__":
    main()
