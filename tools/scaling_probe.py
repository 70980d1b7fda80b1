"""Developer probe: per-rank sweep time of an N-rank strong-scaling run, emulated on
one GPU (PCSB_EMULATE_RANK=N:r: the rank's real layout and kernels, no exchange)."""
import os
import subprocess
import sys

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
code = r'''
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb
cfg = int(sys.argv[1])
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
plan.upload(P, X0)
plan.run(3)
plan.reset()
plan.run(10)
_, s = plan.download()
print(f"{s.sweeps_ms/10:.4f} {s.kernel_ms/10:.4f} {s.sort_ms/10:.4f}")
'''
base = None
for n in (1, 2, 4, 8):
    worst = 0.0
    for r in range(n):  # every rank: the slowest one sets the sweep
        env = dict(os.environ)
        if n > 1:
            env["PCSB_EMULATE_RANK"] = f"{n}:{r}"
        out = subprocess.run([sys.executable, "-c", code, cfg], env=env, capture_output=True,
                             text=True, check=True).stdout.split()
        t = float(out[0])
        worst = max(worst, t)
        print(f"N={n} rank {r}: sweep {out[0]} ms kernel {out[1]} grid {out[2]}", flush=True)
    if base is None:
        base = worst
    print(f"N={n}: slowest rank {worst:.3f} ms -> compute-only speedup {base / worst:.2f}x", flush=True)
