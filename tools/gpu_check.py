"""Developer check on a B200 (not part of the test suite): parity + timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402


def diag(P):
    return float(np.linalg.norm(P.max(0) - P.min(0)))


def section(name):
    print(f"\n=== {name} ===", flush=True)


section("config 1 fp64 vs oracle")
P, X0 = pb.generate_config(1)
prm, c = pb.config_params(1)
t = time.time()
out, s = pb.lop_project(P, X0, prm, precision="fp64")
t1 = time.time() - t
r = O.lop_project(P, X0, prm.kernel.h, prm.kernel.cutoff_multiple, prm.mu, prm.iterations)
err = np.abs(out - r.points).max()
print(f"max|dx|={err:.3e} diag={diag(P):.3f} tol={1e-5*diag(P):.3e} wall={t1:.3f}s", s.iterations_run,
      r.iterations_run, s.interactions_attr, r.interactions_attr, s.interactions_rep,
      r.interactions_rep, s.coincident_pairs, r.coincident_pairs, s.isolated_events,
      r.isolated_events, "sweeps_ms", s.sweeps_ms)

section("plane frozen ratio (test_lop.cpp:119-133)")
D = pb.add_noise(pb.generate_surface("plane", 2000, 11), 0.05, 55)
init = D[::10][:200]
q, s = pb.lop_project(D, init, pb.LopParams(kernel=pb.KernelParams(0.3), mu=0.4))
ratio = np.abs(q[:, 2]).sum() / np.abs(init[:, 2]).sum()
r = O.lop_project(D, init, 0.3, 3.0, 0.4, 30)
print("ratio", repr(ratio), "frozen 0.07335543385137086", "max|dx| vs oracle", np.abs(q - r.points).max())

section("radius queries fp64 / fp32")
for prec in ("fp64", "fp32"):
    Cc = P if prec == "fp64" else P.astype(np.float32).astype(np.float64)
    Q = X0 if prec == "fp64" else X0.astype(np.float32).astype(np.float64)
    off, idx = pb.radius_query_all(Cc, Q, 0.1, precision=prec)
    o2, i2, _ = O.radius_query_all(Cc, Q, 0.1)
    print(prec, "offsets equal", np.array_equal(off, o2), "idx equal", np.array_equal(idx, i2), int(off[-1]))

section("grid sort stability")
keys, order = pb.grid_sort(P, 0.1)
ok_sorted = bool(np.all(np.diff(keys.astype(np.int64)) >= 0))
ties = keys[1:] == keys[:-1]
ok_stable = bool(np.all(order[1:][ties] > order[:-1][ties]))
print("sorted", ok_sorted, "stable", ok_stable)

for cfg, scale in ((3, 0.01), (2, 0.02), (4, 0.01)):
    section(f"config {cfg} @ scale {scale} fp32 vs oracle")
    P, X0 = pb.generate_config(cfg, scale)
    P = P.astype(np.float32).astype(np.float64)
    X0 = X0.astype(np.float32).astype(np.float64)
    prm, c = pb.config_params(cfg)
    # keep neighbour counts comparable to the full config
    hs = c["h"] / np.sqrt(scale) if cfg != 2 else c["h"] / np.sqrt(scale)
    prm, c = pb.config_params(cfg, h=min(hs, 0.3))
    t = time.time()
    out, s = pb.lop_project(P, X0, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    t1 = time.time() - t
    t = time.time()
    r = O.lop_project(P, X0, prm.kernel.h, 4.0, prm.mu, prm.iterations,
                      eta=O.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else O.ETA_INV_CUBE, store_f32=True,
                      wlop=c["wlop"])
    t2 = time.time() - t
    err = np.abs(out - r.points).max()
    print(f"h={prm.kernel.h*4:.4f} max|dx|={err:.3e} tol={1e-5*diag(P):.3e} gpu={t1:.2f}s cpu={t2:.2f}s",
          "attr", s.interactions_attr, r.interactions_attr, "rep", s.interactions_rep,
          r.interactions_rep, "careful", s.careful_points, "iso", s.isolated_events,
          r.isolated_events, "coinc", s.coincident_pairs, r.coincident_pairs)

section("config 3 full, fp32 plan timing")
P, X0 = pb.generate_config(3)
prm, c = pb.config_params(3)
plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
t = time.time()
plan.upload(P, X0)
print("upload+setup wall", time.time() - t)
plan.run(2)
plan.reset()
plan.run(15)
ms = plan.last_run_ms()
out, s = plan.download()
inter = s.interactions_attr + s.interactions_rep
print(f"15 sweeps {ms:.2f} ms -> {inter/ (ms/1e3):.3e} int/s, {15/(ms/1e3):.1f} sweeps/s;",
      "kernel_ms", s.kernel_ms, "sort_ms", s.sort_ms, "careful", s.careful_points,
      "attr/sweep", s.interactions_attr / 15, "rep/sweep", s.interactions_rep / 15,
      "launches", plan.launches())
