"""Developer probe: fp32 queries deferred to the exact fp64 kernel, per config."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
for cfg in [int(a) for a in sys.argv[1:]]:
    P, X0 = pb.generate_config(cfg)
    prm, c = pb.config_params(cfg)
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision=c["precision"])
    plan.upload(P, X0)
    plan.run(6)
    _, s = plan.download()
    print(f"config {cfg}: careful points {s.careful_points} over 6 sweeps, isolated events "
          f"{s.isolated_events}, coincident {s.coincident_pairs}")
    plan.close()
