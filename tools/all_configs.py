"""Developer probe: steady-state throughput of every BASELINE config on one GPU
(3 warm-up sweeps, reset, K timed sweeps, best of 3), fp32 configs 2-5 and the
fp64 config 1, plus config 5 at h in {0.01, 0.02, 0.04}."""
import sys

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

cases = [(1, None, 20), (2, None, 30), (3, None, 15), (4, None, 20), (5, 0.01, 10), (5, 0.02, 10),
         (5, 0.04, 5)]
if len(sys.argv) > 1:  # subset: config numbers
    keep = {int(a) for a in sys.argv[1:]}
    cases = [c for c in cases if c[0] in keep]
print("| config | h | precision | sweeps/s | interactions / sweep | interactions/s | lc/int |")
print("|---|---:|---|---:|---:|---:|---:|")
for cfg, h, k in cases:
    P, X0 = pb.generate_config(cfg)
    prm, c = pb.config_params(cfg, h)
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision=c["precision"])
    plan.upload(P, X0)
    best = None
    for _ in range(3):
        plan.reset()
        plan.run(k)
        _, s = plan.download()
        t = s.sweeps_ms / s.iterations_run
        if best is None or t < best[0]:
            best = (t, s)
    t, s = best
    inter = (s.interactions_attr + s.interactions_rep) / s.iterations_run
    lc = s.lane_candidates / max(1.0, inter * s.iterations_run)
    print(f"| {cfg} | {prm.kernel.support():g} | {c['precision']} | {1e3 / t:.1f} | {inter:.3e} | "
          f"{inter / t * 1e3:.3e} | {lc:.2f} |", flush=True)
    plan.close()
