"""Developer check: WLOP density weights and single sweeps vs the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb
from oracle import oracle as O

P, X0 = pb.generate_config(2, 0.02)
P = P.astype(np.float32).astype(np.float64)
X0 = X0.astype(np.float32).astype(np.float64)
h = 0.3 / 4
vo = O.density_weights(P, h, 4.0)
for prec in ("fp64", "fp32"):
    v = pb.density_weights(P, h, 4.0, precision=prec)
    print(prec, "v rel err", np.abs(v / vo - 1).max())
for wl in (True, False):
    for mu in (0.0, 0.45):
        for it in (1, 5, 30):
            prm = pb.LopParams(kernel=pb.KernelParams(h, 4.0), mu=mu, iterations=it)
            for prec in ("fp64", "fp32"):
                r = O.lop_project(P, X0, h, 4.0, mu, it, eta=O.ETA_NEG_LINEAR, wlop=wl,
                                  store_f32=(prec == "fp32"))
                out, s = pb.lop_project(P, X0, prm, eta="neg_linear", density_weights=wl,
                                        precision=prec)
                e = np.abs(out - r.points).max(1)
                print(f"wlop={wl} mu={mu} it={it} {prec} maxerr={e.max():.3e} "
                      f"n>1e-5={int((e > 1e-5).sum())} careful={s.careful_points} "
                      f"iso {s.isolated_events}/{r.isolated_events} coinc {s.coincident_pairs}/{r.coincident_pairs}")
