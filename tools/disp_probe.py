"""Developer probe: per-sweep displacement statistics (in units of the support)
of one config, to size a skin for a lazily rebuilt projected-set grid."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
P, X0 = pb.generate_config(cfg, 1.0)
prm, c = pb.config_params(cfg)
s = prm.kernel.support()
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
plan.upload(P, X0)
prev = X0.astype(np.float32).astype(np.float64)
acc = np.zeros(len(X0))
for k in range(sweeps):
    plan.run(1)
    out, sm = plan.download()
    d = np.linalg.norm(out - prev, axis=1) / s
    acc += d
    q = np.percentile(d, [50, 99, 99.9, 100])
    print(f"sweep {k + 1}: disp/s p50 {q[0]:.4f} p99 {q[1]:.4f} p99.9 {q[2]:.4f} max {q[3]:.4f} "
          f"(summary {sm.last_max_disp / s:.4f}); cumulative max {acc.max():.3f}", flush=True)
    prev = out
