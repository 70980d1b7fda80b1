"""Generates tests/golden/reference_metrics.npz from the UNMODIFIED reference.

Run where /root/reference exists (oracle/_ref is the reference compiled from its
own sources by `make -C oracle ref`):

    python tests/golden/make_golden_metrics.py

Every output array comes from the reference's own functions on seeded inputs
stored beside them: SpatialIndex::nearest (proj/src/spatial.cpp:119-158),
pcs::deviation (proj/src/metrics.cpp:39-53), pcs::deviation_to_mesh (:115-133)
and point_triangle_distance (:55-113).  The fixture pins the CPU restatement
(oracle/lop_oracle.c) and the B200 kernels bit-for-bit where /root/reference
does not exist.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def cases():
    rng = np.random.default_rng(2024)
    out = {}
    # nearest: random cloud with duplicated points (equal-distance ties), queries
    # inside, on and far outside the cloud
    C = rng.uniform(-1.0, 1.0, (4000, 3))
    C[1500:1600] = C[100:200]                    # exact duplicates -> index tie-break
    Q = np.concatenate([rng.uniform(-1.2, 1.2, (1500, 3)), C[:200],
                        rng.uniform(-50.0, 50.0, (50, 3))])
    out["nn_C"], out["nn_Q"] = C, Q
    # a planar lattice (zero z extent; many equal distances)
    g = np.stack(np.meshgrid(np.arange(40) * 0.025, np.arange(40) * 0.025, [0.0]),
                 -1).reshape(-1, 3)
    qg = np.concatenate([g[::7] + [0.0125, 0.0125, 0.0], g[::11] + [0.0, 0.0, 0.3]])
    out["nn_lattice_C"], out["nn_lattice_Q"] = g, qg
    # deviation: noisy sphere sample vs a denser one (proj/tests/test_metrics.cpp style)
    S = O.ref_generate_surface(1, 3000, 5)
    X = O.ref_add_noise(O.ref_generate_surface(1, 800, 6), 0.01, 7)
    out["dev_cloud"], out["dev_ref"] = X, S
    # mesh: random triangles incl. degenerate ones (repeated vertex, collinear)
    T = rng.uniform(-1.0, 1.0, (80, 9))
    T[5, 6:9] = T[5, 0:3]
    T[6, 3:6] = T[6, 0:3]
    T[6, 6:9] = T[6, 0:3]
    T[7, 6:9] = 0.5 * (T[7, 0:3] + T[7, 3:6])
    P = rng.uniform(-1.5, 1.5, (600, 3))
    out["mesh_T"], out["mesh_P"] = T, P
    return out


def main() -> None:
    O.build(reference=True)
    assert O.ref_available(), "oracle/_ref not built (needs /root/reference)"
    out = cases()
    for k in ("", "_lattice"):
        i, d = O.ref_nearest_all(out[f"nn{k}_C"], out[f"nn{k}_Q"])
        out[f"nn{k}_idx"], out[f"nn{k}_dist"] = i, d
    rep, dist = O.ref_deviation(out["dev_cloud"], out["dev_ref"])
    out["dev_report"], out["dev_dist"] = rep, dist
    rep, dist = O.ref_deviation_to_mesh(out["mesh_P"], out["mesh_T"])
    out["mesh_report"], out["mesh_dist"] = rep, dist
    out["ptri"] = np.array([O.ref_point_triangle_distance(p, out["mesh_T"][t % 80])
                            for t, p in enumerate(out["mesh_P"][:200])])
    np.savez_compressed(os.path.join(HERE, "reference_metrics.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_metrics.npz"), {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
