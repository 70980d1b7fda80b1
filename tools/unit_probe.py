"""Developer probe: sweep time for the full config-3 X0 and for 1/8 of it (the per-GPU
query count of an 8-GPU strong-scaling run), full data cloud."""
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

P, X0 = pb.generate_config(3)
prm, c = pb.config_params(3)
for frac in (1, 8):
    X = X0[: len(X0) // frac]
    plan = pb.LopPlan(prm, eta=c["eta"], precision="fp32")
    plan.upload(P, X)
    plan.run(3)
    plan.reset()
    plan.run(10)
    _, s = plan.download()
    plan.close()
    print(f"X0/{frac}: {s.sweeps_ms/10:.3f} ms/sweep kernel {s.kernel_ms/10:.3f} grid {s.sort_ms/10:.3f}")
