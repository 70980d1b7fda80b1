"""Small LOP/WLOP runs for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of a sweep at smoke size — fast_kernel (attraction and
repulsion passes, fp32), density_kernel (WLOP v_j and w_i), the exact fp64
kernel, the grid build (radix sort incl. the cooperative single-launch sort,
cell tables, pair records) and the deferred-query path.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03365_b200 as pb  # noqa: E402


def r32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    # config 3 shape (LOP, eta = -r), fp32 fused passes + grid rebuilds
    P, X0 = pb.generate_config(3, 0.002)
    prm, c = pb.config_params(3, h=0.2)
    prm.iterations = 2
    out, s = pb.lop_project(r32(P), r32(X0), prm, eta=c["eta"], precision="fp32")
    print("config 3 fp32:", s.iterations_run, s.interactions_attr, s.interactions_rep)
    # config 2 shape (WLOP, outliers -> deferred exact queries)
    P, X0 = pb.generate_config(2, 0.005)
    prm, c = pb.config_params(2, h=0.3)
    prm.iterations = 2
    out, s = pb.lop_project(r32(P), r32(X0), prm, eta=c["eta"], density_weights=True,
                            precision="fp32")
    print("config 2 WLOP fp32:", s.iterations_run, s.interactions_attr, s.careful_points)
    # config 1 shape, fp64 exact path (inverse-cube eta)
    P, X0 = pb.generate_config(1, 0.1)
    prm, _ = pb.config_params(1)
    prm.iterations = 2
    out, s = pb.lop_project(P, X0, prm, precision="fp64")
    print("config 1 fp64:", s.iterations_run, s.interactions_attr)


if __name__ == "__main__":
    main()
