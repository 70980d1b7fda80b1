"""Developer timing/profiling driver: one config, fp32 plan, K sweeps."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--lanes", type=int, nargs="+", default=[4])
ap.add_argument("--sweeps", type=int, default=15)
ap.add_argument("--h", type=float, default=None)
args = ap.parse_args()

P, X0 = pb.generate_config(args.config, args.scale)
prm, c = pb.config_params(args.config, args.h)
for L in args.lanes:
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32",
                      lanes_per_point=L)
    t = time.time()
    plan.upload(P, X0)
    up = time.time() - t
    plan.run(args.sweeps)
    ms = plan.last_run_ms()
    out, s = plan.download()
    inter = s.interactions_attr + s.interactions_rep
    print(f"cfg{args.config} L={L} upload {up:.2f}s  {args.sweeps} sweeps {ms:.2f} ms -> "
          f"{inter / (ms / 1e3):.3e} int/s {args.sweeps / (ms / 1e3):.1f} sweeps/s kernel_ms "
          f"{s.kernel_ms:.2f} sort_ms {s.sort_ms:.2f} careful {s.careful_points} "
          f"int/sweep {inter / args.sweeps:.3e} dens {s.density_pairs} lc/int {s.lane_candidates / max(1, inter):.3f}", flush=True)
    plan.close()
