"""Developer check: config-2 sweep-1 counts and density weights: oracle vs single vs sharded."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2401_03365_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_sharded import _sharded, _single  # noqa: E402

cfg, scale, nr = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
P, X0 = pb.generate_config(cfg, scale)
P = P.astype(np.float32).astype(np.float64)
X0 = X0.astype(np.float32).astype(np.float64)
prm, c = pb.config_params(cfg)
prm.iterations = 1
kw = dict(eta=c["eta"], density_weights=c["wlop"], precision="fp32")
ref, sr = _single(P, X0, prm, **kw)
outs = _sharded(P, X0, prm, nr, **kw)
eta = O.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else O.ETA_INV_CUBE
r = O.lop_project(P, X0, prm.kernel.h, 4.0, c["mu"], 1, eta=eta, wlop=c["wlop"], store_f32=True)
print("attr oracle/single/shard", r.interactions_attr, sr.interactions_attr, outs[0][1].interactions_attr)
print("rep  oracle/single/shard", r.interactions_rep, sr.interactions_rep, outs[0][1].interactions_rep)
wo = O.density_weights(X0, prm.kernel.h, 4.0)
wg = pb.density_weights(X0, prm.kernel.h, 4.0, precision="fp32") if hasattr(pb, "density_weights") else None
print("density facility vs oracle max rel", np.abs(wg / wo - 1).max() if wg is not None else None)
es = np.abs(ref - r.points).max(1)
eh = np.abs(outs[0][0] - r.points).max(1)
print("single vs oracle: max", es.max(), "n>1e-6", (es > 1e-6).sum(), " shard vs oracle: max", eh.max(), "n>1e-6", (eh > 1e-6).sum())
bad = np.flatnonzero(eh > 1e-6)[:10]
print("bad idx", bad, "X0 of first bad", X0[bad[:3]] if len(bad) else None)
