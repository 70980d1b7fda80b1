"""Developer probe: steady sweep time of the current process's (emulated) rank,
config 3 (3 warm-up sweeps, reset, 10 timed) — the inner step of scaling_probe.py."""
import sys

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
plan.upload(P, X0)
plan.run(3)
plan.reset()
plan.run(10)
_, s = plan.download()
inter = s.interactions_attr + s.interactions_rep
print(f"sweep {s.sweeps_ms / 10:.4f} ms kernel {s.kernel_ms / 10:.4f} grid {s.sort_ms / 10:.4f} "
      f"attr/sweep {s.interactions_attr / 10:.4e} rep/sweep {s.interactions_rep / 10:.4e} "
      f"lc/int {s.lane_candidates / max(1, inter):.3f}")
