"""Developer probe: per-phase sweep times (PCSB_DEBUG_TIMES) for config 3."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
P, X0 = pb.generate_config(3)
prm, c = pb.config_params(3)
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 0
plan = pb.LopPlan(prm, eta=c["eta"], precision="fp32", lanes_per_point=lanes)
plan.upload(P, X0)
plan.run(4)
plan.close()
