"""Developer A/B probe: for each env variant, run the config's plan (3 warm-up
sweeps, reset, K timed sweeps) REPS times in one process per variant and report
the best sweep time — robust to box noise.

    python tools/ab_probe.py CONFIG SWEEPS REPS 'ENV=1 ENV2=x' 'ENV=0' ...
"""
import os
import subprocess
import sys

code = r'''
import sys
sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb
cfg, k, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
plan.upload(P, X0)
best = None
for r in range(reps):
    plan.reset()
    plan.run(k)
    _, s = plan.download()
    t = s.sweeps_ms / k
    if best is None or t < best[0]:
        best = (t, s)
t, s = best
inter = (s.interactions_attr + s.interactions_rep) / k
print(f"{t:.4f} ms/sweep {inter / t * 1e3:.4e} int/s lc/int {s.lane_candidates / max(1, k * inter):.3f}")
'''
cfg, k, reps = sys.argv[1], sys.argv[2], sys.argv[3]
for variant in sys.argv[4:]:
    env = dict(os.environ)
    for kv in variant.split():
        a, b = kv.split("=", 1)
        env[a] = b
    out = subprocess.run([sys.executable, "-c", code, cfg, k, reps], env=env, capture_output=True,
                         text=True).stdout.strip()
    print(f"cfg {cfg} [{variant}] {out}", flush=True)
