"""Developer probe: per-phase sweep times (PCSB_DEBUG_TIMES) for a config."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
cfg = int(sys.argv[1])
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision=c["precision"])
plan.upload(P, X0)
plan.run(3)
plan.reset()
plan.run(6)
print("launches", plan.launches())
plan.close()
