"""Developer probe: sweep time with and without CUDA-graph replay (configs 1, 2, 3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03365_b200 as pb  # noqa: E402

for cfg, k, prec in ((1, 40, "fp64"), (2, 40, "fp32"), (3, 17, "fp32")):
    P, X0 = pb.generate_config(cfg)
    prm, c = pb.config_params(cfg)
    prm.convergence_tol = 1e-30
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision=prec)
    plan.upload(P, X0)
    for on in (False, True, False, True):
        plan.set_graphs(on)
        best = None
        for r in range(3):
            plan.reset()
            l0, g0 = plan.launches(), plan.graph_launches()
            plan.run(k)
            _, s = plan.download()
            t = s.sweeps_ms / k
            if best is None or t < best[0]:
                best = (t, (plan.launches() - l0) / k, plan.graph_launches() - g0, s.iterations_run,
                        s.interactions_attr)
        print(f"cfg {cfg} graphs={int(on)}: {best[0]:.4f} ms/sweep ({1e3 / best[0]:.0f} sweeps/s), "
              f"{best[1]:.1f} kernels/sweep, {best[2]} graph launches, iterations {best[3]}, "
              f"attr {best[4]}", flush=True)
    plan.close()
