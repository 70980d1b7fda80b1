"""Developer check: per-sweep agreement of loopback-sharded vs single-rank runs."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2401_03365_b200 as pb  # noqa: E402
from test_gpu_sharded import _sharded, _single  # noqa: E402

cfg, scale, nr = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
P, X0 = pb.generate_config(cfg, scale)
for it in (1, 2, 3, 4):
    prm, c = pb.config_params(cfg)
    prm.iterations = it
    kw = dict(eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    ref, sr = _single(P, X0, prm, **kw)
    outs = _sharded(P, X0, prm, nr, **kw)
    X, s = outs[0]
    d = np.abs(X - ref).max(1)
    print(f"it={it} attr {s.interactions_attr}/{sr.interactions_attr} rep {s.interactions_rep}/{sr.interactions_rep} "
          f"dens {s.density_pairs}/{sr.density_pairs} careful {s.careful_points}/{sr.careful_points} "
          f"maxdiff {d.max():.3e} n>1e-6 {(d > 1e-6).sum()}")
