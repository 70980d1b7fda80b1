"""Developer probe: one plan upload of a config (its data-grid radix sort is the largest sort)."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
plan.upload(P, X0)
plan.run(1)
plan.close()
print("ok", P.shape, X0.shape)
