"""Developer probe: attraction-only vs full sweep cost on a config (mu = 0 disables repulsion)."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P, X0 = pb.generate_config(cfg)
for mu in (None, 0.0):
    prm, c = pb.config_params(cfg)
    if mu is not None:
        prm.mu = mu
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    plan.upload(P, X0)
    plan.run(3)
    plan.reset()
    plan.run(10)
    _, s = plan.download()
    print(f"mu={prm.mu}: kernel {s.kernel_ms/10:.3f} ms/sweep grid {s.sort_ms/10:.3f} attr/sweep {s.interactions_attr/10:.3e} "
          f"rep/sweep {s.interactions_rep/10:.3e} lc/int {s.lane_candidates/max(1,s.interactions_attr+s.interactions_rep):.3f}")
