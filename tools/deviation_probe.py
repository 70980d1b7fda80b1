"""Developer probe: deviation metric (nearest reference point of every projected
point) on config 3 — B200 (pcs_deviation through the C ABI, host buffers, warm
call) vs the reference's pcs::deviation on all host cores (oracle/_ref)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
P, X0 = pb.generate_config(3, scale)
rng = np.random.default_rng(1)
X = X0 + rng.normal(scale=0.002, size=X0.shape)
pb.deviation(X[:1000], P[:10000], device=0)  # context + module load
ts = []
for _ in range(3):
    t = time.perf_counter()
    r = pb.deviation(X, P, keep_distances=True, device=0)
    ts.append(time.perf_counter() - t)
print(f"B200 deviation: P={P.shape[0]} X={X.shape[0]} wall {min(ts)*1e3:.1f} ms (best of 3) "
      f"mean {r.mean_distance:.6e} rms {r.std_deviation:.6e} max {r.max_distance:.6e}", flush=True)
if O.ref_available():
    t = time.perf_counter()
    rr, rd = O.ref_deviation(X, P)
    tr = time.perf_counter() - t
    exact = bool(np.array_equal(rd, r.distances)) and list(rr) == [r.n, r.mean_distance,
                                                                   r.std_deviation, r.max_distance]
    print(f"reference deviation ({os.cpu_count()} host threads, kd-tree build included): "
          f"{tr*1e3:.1f} ms; bit-exact report and distances: {exact}", flush=True)
