"""Developer check: per-sweep parity from the GPU's own iterate X^k."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb
from oracle import oracle as O

for cfg, scale, hh in ((2, 0.02, 0.3), (3, 0.01, 0.2), (4, 0.01, 0.3), (5, 0.001, 0.3)):
    P, X0 = pb.generate_config(cfg, scale)
    P = P.astype(np.float32).astype(np.float64)
    X0 = X0.astype(np.float32).astype(np.float64)
    prm, c = pb.config_params(cfg, h=hh)
    h = prm.kernel.h
    eta = O.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else O.ETA_INV_CUBE
    diag = np.linalg.norm(P.max(0) - P.min(0))
    for k in (0, 10, 25):
        if k:
            prm.iterations = k
            Xk, _ = pb.lop_project(P, X0, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
        else:
            Xk = X0
        for s in (1, 2):
            prm.iterations = s
            out, st = pb.lop_project(P, Xk, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
            r = O.lop_project(P, Xk, h, 4.0, c["mu"], s, eta=eta, wlop=c["wlop"], store_f32=True)
            e = np.abs(out - r.points).max(1)
            print(f"cfg{cfg} from X^{k} +{s} sweeps: max={e.max():.3e} (tol {1e-5*diag:.1e}) "
                  f"n>tol={(e > 1e-5*diag).sum()} n>1e-6={(e>1e-6).sum()} careful={st.careful_points} "
                  f"attr {st.interactions_attr}/{r.interactions_attr} rep {st.interactions_rep}/{r.interactions_rep} "
                  f"coinc {st.coincident_pairs}/{r.coincident_pairs} iso {st.isolated_events}/{r.isolated_events}",
                  flush=True)
