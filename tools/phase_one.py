"""Developer probe: per-phase sweep times (PCSB_DEBUG_TIMES, dev builds) of one
config, optionally one emulated rank (PCSB_EMULATE_RANK=N:r)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
plan.upload(P, X0)
plan.run(3)
plan.reset()
plan.run(6)
_, s = plan.download()
inter = s.interactions_attr + s.interactions_rep
print(f"cfg {cfg}: {s.sweeps_ms / 6:.4f} ms/sweep, kernel {s.kernel_ms / 6:.4f} ms, interactions/sweep "
      f"{inter / 6:.4e}, lc/int {s.lane_candidates / max(1, inter):.3f}")
