"""Developer probe: sweep time and candidates per interaction vs lanes per query
(LopDesc.lanes_per_point: L lanes per query, Q = 32/L queries per staged group).

    python tools/lanes_probe.py CONFIG [SWEEPS] [REPS] [L ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1])
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
lanes = [int(v) for v in sys.argv[4:]] or [4, 8, 2]
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
for L in lanes:
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32",
                      lanes_per_point=L)
    plan.upload(P, X0)
    best = None
    for r in range(reps):
        plan.reset()
        plan.run(k)
        _, s = plan.download()
        t = s.sweeps_ms / k
        if best is None or t < best[0]:
            best = (t, s)
    t, s = best
    inter = (s.interactions_attr + s.interactions_rep) / k
    print(f"cfg {cfg} L={L}: {t:.4f} ms/sweep {inter / t * 1e3:.4e} int/s "
          f"lc/int {s.lane_candidates / max(1, k * inter):.3f}", flush=True)
    plan.close()
