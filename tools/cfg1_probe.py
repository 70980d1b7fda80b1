"""Developer probe: config 1 (fp64 exact path) sweep time, kernel launches per sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03365_b200 as pb  # noqa: E402

P, X0 = pb.generate_config(1)
prm, c = pb.config_params(1)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
plan = pb.LopPlan(prm, precision="fp64")
plan.upload(P, X0)
best = None
for r in range(5):
    plan.reset()
    l0 = plan.launches()
    t = time.perf_counter()
    plan.run(k)
    wall = time.perf_counter() - t
    _, s = plan.download()
    ms = s.sweeps_ms / k
    if best is None or ms < best[0]:
        best = (ms, wall / k * 1e3, (plan.launches() - l0) / k)
print(f"config 1: {best[0]:.4f} ms/sweep (device), {best[1]:.4f} ms/sweep (host wall), "
      f"{1e3 / best[0]:.0f} sweeps/s, {best[2]:.1f} launches/sweep")
