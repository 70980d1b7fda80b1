"""Developer probe: per-sweep max displacement of each config (drift bound sizing)."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
for cfg in (3, 4, 5, 2):
    P, X0 = pb.generate_config(cfg, 1.0 if cfg != 5 else 0.2)
    prm, c = pb.config_params(cfg)
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    plan.upload(P, X0)
    d = []
    for k in range(prm.iterations):
        plan.run(1)
        _, s = plan.download()
        d.append(s.last_max_disp)
    plan.close()
    print(f"cfg{cfg} support {prm.kernel.support():.3f} max disp per sweep / support:",
          " ".join(f"{v / prm.kernel.support():.3f}" for v in d))
