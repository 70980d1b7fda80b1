#!/usr/bin/env python3
"""Benchmark of the B200 LOP/WLOP hot path (BASELINE.json metric).

Workload (default): BASELINE.json configs[2] — LOP on the bumpy height field,
P = 10,000,000 data points, X0 = 1,000,000 (seeded subset), h = 0.02 (support),
mu = 0.4, eta(r) = -r, fp32 — the north star's "10M-point config", sharded over
1/2/4/8 GPUs (strong scaling).  A step is one LOP sweep (grid rebuild + fused
per-point kernel + deferred exact queries + [all-gather] + convergence).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

For N > 1 the driver launches one process per GPU with torch.distributed.run;
the plan joins an NCCL clique and all-gathers X every sweep.

The timed region (value) runs K sweeps with P and X0 already resident in HBM,
bracketed by a barrier and a device synchronize, timed with CUDA events on the
plan's stream, max over ranks.  `e2e` is the same metric through the public
API with host buffers (upload, data grid, K sweeps, download) — wall clock.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

WORKLOADS = {
    1: "config1: LOP noisy unit sphere, P=20k, X0=2k, h=0.1, mu=0.45, eta=1/(3r^3), fp64",
    2: "config2: WLOP torus R=1 r=0.3 + 5% outliers, P=1M, X0=100k, h=0.05, mu=0.45, eta=-r, fp32",
    3: "config3: LOP height field z=0.1 sin8x cos8y, P=10M, X0=1M, h=0.02, mu=0.4, eta=-r, fp32",
    4: "config4: WLOP density sphere ~e^{3.9z}, P=4M, X0=400k, h=0.03, mu=0.45, eta=-r, fp32",
    5: "config5: LOP 8 ellipsoids, P=50M, X0=5M, h=0.02, mu=0.45, eta=1/(3r^3), fp32",
}


# Parameters of the five configurations (h = support radius -> KernelParams{h/4, 4});
# the same table as paper_2401_03365_b200.CONFIGS, repeated here so that the
# reference arm does not import the product package.
CONFIGS = {
    1: dict(h=0.1, mu=0.45, eta="inv_cube", wlop=False, iterations=20, precision="fp64"),
    2: dict(h=0.05, mu=0.45, eta="neg_linear", wlop=True, iterations=30, precision="fp32"),
    3: dict(h=0.02, mu=0.40, eta="neg_linear", wlop=False, iterations=15, precision="fp32"),
    4: dict(h=0.03, mu=0.45, eta="neg_linear", wlop=True, iterations=20, precision="fp32"),
    5: dict(h=0.02, mu=0.45, eta="inv_cube", wlop=False, iterations=10, precision="fp32"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------
# clocks during the timed region (NVML sampled from a thread)
# ------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.0005):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.period = period_s
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            log("NVML unavailable:", e)
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
            # the timed region is short (~70 ms on the default config): make sure the
            # sampler is running before it starts
            t0 = time.time()
            while not self.samples and time.time() - t0 < 1.0:
                time.sleep(0.0005)

    def stop(self) -> dict:
        if not self._thr:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        self._stop.set()
        self._thr.join()
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": reasons}


# ------------------------------------------------------------------------------
# roofline denominators
# ------------------------------------------------------------------------------
def sfu_peak(sm_mhz: float, sms: int = 148) -> dict:
    """Interactions/s bound of the fused kernel.

    Per interaction the kernel needs 2 MUFU ops (ex2 for theta, rsqrt for 1/d);
    sm_100 issues 16 MUFU results per SM per clock, so the bound is
    8 interactions / SM / clock.  profiles/pipe_peaks.json, when
    present, holds the MUFU rate measured on this pool's B200s.
    """
    per_sm_clk = 8.0
    src = "derived: 16 MUFU/SM/clk (sm_100) / 2 MUFU per interaction x 148 SMs x clock"
    p = os.path.join(HERE, "profiles", "pipe_peaks.json")
    if os.path.exists(p):
        try:
            pk = json.load(open(p))
            per_sm_clk = pk["mufu_per_sm_clk"] / 2.0
            src = f"measured MUFU rate {pk['mufu_per_sm_clk']:.2f}/SM/clk (profiles/pipe_peaks.json) / 2"
        except Exception:
            pass
    return {"per_sm_clk": per_sm_clk, "peak": per_sm_clk * sms * sm_mhz * 1e6, "source": src}


# ------------------------------------------------------------------------------
# CPU baseline: the reference's own lop_project on the host cores
# ------------------------------------------------------------------------------
def cpu_baseline(cfg: int, P: np.ndarray, X0: np.ndarray, c: dict, repeats: int = 5,
                 sweeps: int = 11) -> dict:
    """The reference's own CPU path on a bounded, seeded sample of the workload.

    LOP configs run oracle/_ref — the unmodified reference compiled from
    /root/reference (kind "reference"); for eta = -r the same objects with
    lop.cpp's |eta'| call bound to 1 (oracle/ref_etar_wrap.cpp), so the
    arithmetic per interaction is the configuration's.  WLOP configs (no
    reference implementation) run the oracle port (kind "port").

    pcs::lop_project builds the kd-tree of the FULL data cloud inside the call
    (lop.cpp:24), seconds at 10M points.  The sweep rate is therefore the
    difference of a `sweeps`-sweep call and a 1-sweep call on the same sample
    (the index build cancels), median of `repeats`; the interactions of sweeps
    2..K are counted by the oracle port on the same sample (not timed)."""
    from oracle import oracle as O

    nthreads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(nthreads))
    rng = np.random.default_rng(12345)
    frac = 0.02 if X0.shape[0] >= 100000 else 1.0
    nsub = max(1, int(X0.shape[0] * frac))
    sub = np.sort(rng.choice(X0.shape[0], nsub, replace=False))
    Xs = np.ascontiguousarray(X0[sub])
    h, cut, mu = c["h"] / 4.0, 4.0, c["mu"]
    eta_kind = O.ETA_NEG_LINEAR if c["eta"] == "neg_linear" else O.ETA_INV_CUBE
    use_ref = O.ref_available() and not c["wlop"]
    c1 = O.lop_project(P, Xs, h, cut, mu, 1, eta=eta_kind, wlop=c["wlop"])
    cK = O.lop_project(P, Xs, h, cut, mu, sweeps, eta=eta_kind, wlop=c["wlop"])
    inter = (cK.interactions_attr + cK.interactions_rep) - (c1.interactions_attr + c1.interactions_rep)

    def call(k):
        t = time.perf_counter()
        if use_ref:
            O.ref_lop_project(P, Xs, h, cut, mu, k, eta=eta_kind)
        else:
            O.lop_project(P, Xs, h, cut, mu, k, eta=eta_kind, wlop=c["wlop"])
        return time.perf_counter() - t

    t1s, tKs = [], []
    for _ in range(repeats):  # interleaved: drifts of the host affect both alike
        t1s.append(call(1))
        tKs.append(call(sweeps))
    t1, tK = statistics.median(t1s), statistics.median(tKs)
    t_sweeps = max(1e-9, tK - t1)
    lib = "oracle/_ref/libpcs_ref_etar.so" if eta_kind == O.ETA_NEG_LINEAR else "oracle/_ref/libpcs_ref.so"
    if use_ref:
        kind = "reference"
        what = (f"reference pcs::lop_project ({lib}, built from /root/reference"
                f"{'; lop.cpp with |eta_prime| = 1 for eta = -r' if eta_kind == O.ETA_NEG_LINEAR else ''}) "
                f"on a seeded {nsub}-point subset of X0 against the full P ({P.shape[0]} pts), "
                f"{c['eta']} eta as configured: time of a {sweeps}-sweep call minus a 1-sweep call "
                f"(the in-call kd-tree build of P cancels), median of {repeats}; interactions of "
                f"sweeps 2..{sweeps} ({inter}) counted by the oracle port")
    else:
        kind = "port"
        what = (f"oracle port (oracle/lop_oracle.c, OpenMP; the reference has no WLOP) on a seeded "
                f"{nsub}-point subset of X0 against the full P ({P.shape[0]} pts): {sweeps}-sweep "
                f"call minus 1-sweep call, median of {repeats}")
    per = [max(1e-9, b - a) for a, b in zip(t1s, tKs)]
    return {"value": inter / t_sweeps, "unit": "interactions/s", "cores": int(os.environ.get(
        "OMP_NUM_THREADS", nthreads)), "kind": kind, "sample": what,
        "sample_interactions": int(inter), "sample_seconds": t_sweeps,
        "sweeps_timed": sweeps - 1, "repeats": repeats,
        "rates_per_repeat": [inter / t for t in per],
        "seconds_per_sweep": t_sweeps / (sweeps - 1), "call_seconds": {"1": t1s, str(sweeps): tKs}}


# ------------------------------------------------------------------------------
def self_launch(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: re-executes itself as N ranks
    (one process per GPU) under torch.distributed.run, exactly as the driver
    launches it; fails loudly when fewer than N GPUs are visible."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        log(f"error: --gpus {n} requested but {have} CUDA device(s) are visible")
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    log("launching:", " ".join(cmd))
    os.execv(sys.executable, cmd)
    return 0  # not reached


def bench_mls(args):
    """SURVEY 8(f) row 1 on one B200: smooth_cloud (proj/src/mls.cpp:75-93) of a
    noisy sphere (the reference's bench surface, proj/src/bench.cpp:40-87 via the
    restated generator), h = 0.01.  value = points / device time of the two
    launches (CUDA events inside the library); e2e = the same call's wall time
    with host buffers (upload, index build, launches, download).  The CPU
    baseline is the oracle port of the reference's per-point projection on a
    20000-point sample with all host threads."""
    import ctypes as C
    import paper_2401_03365_b200 as pb
    from paper_2401_03365_b200 import _lib as L
    n, deg, h = args.mls_points, args.mls_degree, 0.01
    P = pb.add_noise(pb.generate_surface("sphere", n, 7), 0.002, 8)
    prm = pb.MlsParams(kernel=pb.KernelParams(h), degree=deg)
    pb.smooth_cloud(P[:1000], prm)
    dev_ms, walls = [], []
    mon = ClockSampler(0)
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            mon.start()
        t = time.perf_counter()
        out, res = pb.smooth_cloud(P, prm)
        wall = time.perf_counter() - t
        a, b = C.c_double(), C.c_double()
        L.lib().pcs_mls_last_device_ms(C.byref(a), C.byref(b))
        if i >= args.warmup:
            dev_ms.append((a.value, b.value))
            walls.append(wall)
    clocks = mon.stop()
    plane = float(np.median([d[0] for d in dev_ms]))
    poly = float(np.median([d[1] for d in dev_ms]))
    wall = float(np.median(walls))
    line = {
        "metric": "MLS projected points/sec (smooth_cloud)", "value": n / ((plane + poly) * 1e-3),
        "unit": "points/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": plane + poly, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded host generator)",
        "config": {"workload": f"MLS smooth_cloud: noisy unit sphere, {n} points, h = {h} "
                               f"(support {3 * h}), degree {deg}",
                   "l2": "the cloud (32 MB as double4) fits L2; every step re-uploads and "
                         "re-indexes it"},
        "device_ms": {"plane_fit_launch": plane, "polynomial_launch": poly},
        "mean_plane_iterations": float(res.iterations.mean()),
        "e2e": {"value": n / wall, "unit": "points/s", "wall_s": wall,
                "h2d_bytes_per_step": int(P.nbytes), "d2h_bytes_per_step": int(out.nbytes + 8 * n),
                "api": "pcs_mls_smooth_outcomes (C ABI) with host buffers"},
        "gpu_launches": 2 * args.steps, "clocks": clocks,
        "roofline": None,
        "roofline_note": "instruction-issue bound (ncu: plane launch issue active 71%), see "
                         "DESIGN.md 5d and profiles/r02_mls_kernel_ncu.json",
    }
    if not args.no_cpu:
        from oracle import oracle as O
        sub = np.random.default_rng(0).choice(n, min(n, 20000), replace=False)
        t = time.perf_counter()
        r = O.mls_project(P, P[sub], h, degree=deg)
        tc = time.perf_counter() - t
        line["cpu_baseline"] = {"value": sub.size / tc, "unit": "points/s", "cores": os.cpu_count(),
                                "kind": "port",
                                "sample": f"oracle orc_mls_project on {sub.size} seeded points of the "
                                          f"same cloud, all host threads"}
        line["max_abs_dev_vs_oracle"] = float(np.abs(out[sub] - r["projected"]).max())
    print(json.dumps(line), flush=True)
    return 0


def bench_rows(args):
    """SURVEY 8(f) rows 2 and 3 on one B200, config-3 clouds, through the C ABI
    with host buffers (value = e2e: these operators have no device-resident
    entry point).  deviation: pcs::deviation (proj/src/metrics.cpp:39-53) of
    1M perturbed projected points against the 10M data points; io: XYZ text of
    the 10M-point cloud written and parsed back (proj/src/io.cpp).  The CPU
    baseline is the reference itself (oracle/_ref) on the same inputs
    (deviation) or on a 30% sample of the cloud (io, its IO is single-threaded)."""
    import paper_2401_03365_b200 as pb
    from oracle import oracle as O
    P, X0 = pb.generate_config(3)
    mon = ClockSampler(0)
    if args.workload == "deviation":
        X = X0 + np.random.default_rng(1).normal(scale=0.002, size=X0.shape)
        pb.deviation(X[:1000], P[:10000], device=0)
        walls = []
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                mon.start()
            t = time.perf_counter()
            r = pb.deviation(X, P, keep_distances=True, device=0)
            if i >= args.warmup:
                walls.append(time.perf_counter() - t)
        clocks = mon.stop()
        wall = float(np.median(walls))
        line = {"metric": "deviation queries/sec (nearest data point of every projected point)",
                "value": X.shape[0] / wall, "unit": "queries/s", "ms_per_step": wall * 1e3,
                "config": {"workload": f"deviation: {X.shape[0]} projected points vs {P.shape[0]} "
                                       f"data points (config 3 clouds), fp64, bit-exact distances"},
                "e2e": {"value": X.shape[0] / wall, "unit": "queries/s", "wall_s": wall,
                        "h2d_bytes_per_step": int(P.nbytes + X.nbytes),
                        "d2h_bytes_per_step": int(8 * X.shape[0]),
                        "api": "pcs_deviation (C ABI) with host buffers"},
                "roofline_note": "latency/divergence bound walk (DESIGN.md 5a); the call is "
                                 "dominated by the 240 MB host-to-device copy of the data cloud"}
        if not args.no_cpu and O.ref_available():
            t = time.perf_counter()
            rr, rd = O.ref_deviation(X, P)
            tc = time.perf_counter() - t
            line["cpu_baseline"] = {"value": X.shape[0] / tc, "unit": "queries/s",
                                    "cores": os.cpu_count(), "kind": "reference",
                                    "sample": "pcs::deviation (oracle/_ref) on the same inputs, "
                                              "kd-tree build included"}
            line["bit_exact_vs_reference"] = bool(np.array_equal(rd, r.distances))
    else:
        # the C ABI as a C caller uses it in steady state: caller-owned buffers,
        # reused across calls (the text buffer sized by the 25-character bound per
        # coordinate); the Python mirror's format_cloud adds a copy into `bytes`
        import ctypes as C
        from paper_2401_03365_b200 import _lib as L
        from paper_2401_03365_b200.lop import make_desc, LopParams
        pb.format_cloud(P[:1000], device=0)
        n = P.shape[0]
        d = make_desc(LopParams(), device=0)
        cap = 80 * n + 1024
        tbuf = np.empty(cap, dtype=np.uint8)
        back = np.empty((n + 8, 3), dtype=np.float64)
        tptr = C.cast(tbuf.ctypes.data, C.c_char_p)
        dp = C.POINTER(C.c_double)
        tlen, nback = C.c_uint64(0), C.c_uint64(0)
        err = L.ParseErrorC()
        tw, tr = [], []
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                mon.start()
            t = time.perf_counter()
            st = L.lib().pcs_format_cloud(C.byref(d), P.ctypes.data_as(dp), n, 0, tptr, cap,
                                          C.byref(tlen))
            t1 = time.perf_counter()
            st2 = L.lib().pcs_parse_cloud(C.byref(d), tptr, tlen.value, 0, back.ctypes.data_as(dp),
                                          back.shape[0], C.byref(nback), C.byref(err))
            t2 = time.perf_counter()
            if st != 0 or st2 != 0 or nback.value != n:
                raise RuntimeError(f"cloud IO failed: {st} {st2} {nback.value}")
            if i >= args.warmup:
                tw.append(t1 - t)
                tr.append(t2 - t1)
        text = tbuf[: tlen.value].tobytes()
        back = back[:n]
        clocks = mon.stop()
        w, r_ = float(np.median(tw)), float(np.median(tr))
        nbytes = len(text)
        line = {"metric": "cloud text IO bytes/sec (XYZ write + read)",
                "value": 2 * nbytes / (w + r_), "unit": "bytes/s", "ms_per_step": (w + r_) * 1e3,
                "config": {"workload": f"XYZ text of the config-3 data cloud: {P.shape[0]} points, "
                                       f"{nbytes / 1e6:.0f} MB; shortest round-trip digits, "
                                       f"byte-identical to the reference"},
                "write_s": w, "read_s": r_,
                "e2e": {"value": 2 * nbytes / (w + r_), "unit": "bytes/s", "wall_s": w + r_,
                        "h2d_bytes_per_step": int(P.nbytes + nbytes),
                        "d2h_bytes_per_step": int(P.nbytes + nbytes),
                        "api": "pcs_format_cloud + pcs_parse_cloud (C ABI) with host buffers"},
                "round_trip_bit_exact": bool(np.array_equal(back.view(np.uint64), P.view(np.uint64))),
                "roofline_note": "host-device staging of the text bound (DESIGN.md 5c): device "
                                 "kernels are ~7 ms of the call"}
        if not args.no_cpu and O.ref_available():
            Ps = P[: int(0.3 * P.shape[0])]
            t = time.perf_counter()
            rtext = O.ref_format_cloud(Ps, 0)
            t1 = time.perf_counter()
            rback, err = O.ref_parse_cloud(rtext, 0)
            t2 = time.perf_counter()
            line["cpu_baseline"] = {"value": 2 * len(rtext) / (t2 - t), "unit": "bytes/s", "cores": 1,
                                    "kind": "reference",
                                    "sample": f"write_cloud_stream + read_cloud_stream (oracle/_ref) "
                                              f"on the first {Ps.shape[0]} points"}
            line["identical_bytes_on_sample"] = bool(text[: len(rtext)] == rtext) and err is None
    line.update({"n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                 "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                 "data": "synthetic (seeded host generator, BASELINE.md §4)", "clocks": clocks,
                 "roofline": None})
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=15)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--workload", choices=["lop", "mls", "deviation", "io"], default="lop",
                    help="lop: the BASELINE.json metric (default); the others are the SURVEY "
                         "8(f) rows on one GPU — mls: smooth_cloud points/s on a synthetic "
                         "sphere; deviation: nearest-neighbour metric of 1M projected vs 10M "
                         "data points; io: XYZ text write + read of the 10M-point cloud")
    ap.add_argument("--mls-points", type=int, default=1_000_000)
    ap.add_argument("--mls-degree", type=int, default=2)
    args = ap.parse_args()
    if args.workload == "mls":
        return bench_mls(args)
    if args.workload in ("deviation", "io"):
        return bench_rows(args)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        return self_launch(args.gpus)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE")
    ngpu = world

    cfg = args.config
    c = dict(CONFIGS[cfg])
    precision = c["precision"]

    # ---------------- reference arm ----------------
    if args.impl == "reference":
        # the reference's own CPU path only: inputs come from the oracle's restated
        # generator (the same draws), so this process never loads the product library
        if rank != 0:
            return 0
        from oracle import oracle as O
        t0 = time.perf_counter()
        P, X0 = O.generate_config(cfg)
        if precision == "fp32":
            P = P.astype(np.float32).astype(np.float64)
            X0 = X0.astype(np.float32).astype(np.float64)
        cb = cpu_baseline(cfg, P, X0, c, repeats=5)
        wall = time.perf_counter() - t0
        try:  # evidence: the product library is not mapped in this process
            maps = open("/proc/self/maps").read()
            loaded = sorted({ln.split()[-1] for ln in maps.splitlines()
                             if ln.endswith(".so") and ("/oracle/" in ln or "libpcs" in ln)})
        except OSError:
            loaded = None
        line = {
            "impl": "reference", "libraries_mapped": loaded, "metric": "neighbour interactions/sec (LOP sweep)",
            "value": cb["value"], "unit": "interactions/s", "n_gpus": ngpu,
            "steps": cb["sweeps_timed"], "warmup": 1, "repeats": cb["repeats"],
            "ms_per_step": cb["seconds_per_sweep"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded host generator, BASELINE.md §4)",
            "config": {"workload": WORKLOADS[cfg], "sample": cb["sample"],
                       "note": f"--steps {args.steps} --warmup {args.warmup} requested; a step "
                               f"here is one sweep of the bounded sample (steps = sweeps timed "
                               f"per repeat: a {cb['sweeps_timed'] + 1}-sweep call minus a "
                               f"1-sweep call)"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "rates_per_repeat": cb["rates_per_repeat"],
            "timed_region_s": sum(cb["call_seconds"]["1"]) + sum(
                cb["call_seconds"][str(cb["sweeps_timed"] + 1)]),
            "wall_s": wall,
            "e2e": {"value": cb["value"], "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0

    import paper_2401_03365_b200 as pb
    params, c = pb.config_params(cfg)

    # ---------------- B200 arm ----------------
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(0)
    dev = local_rank if world > 1 else 0

    t0 = time.time()
    P, X0 = pb.generate_config(cfg)
    log(f"[rank {rank}] generated config {cfg}: P={P.shape[0]} X0={X0.shape[0]} "
        f"in {time.time() - t0:.1f}s")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def make_plan():
        plan = pb.LopPlan(params, eta=c["eta"], density_weights=c["wlop"], precision=precision,
                          device=dev, lanes_per_point=args.lanes)
        if world > 1:
            uid = [pb.LopPlan.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            plan.set_comm(uid[0], world, rank)
        return plan

    plan = make_plan()
    t = time.time()
    plan.upload(P, X0)
    log(f"[rank {rank}] upload + data grid {time.time() - t:.2f}s")

    # warm-up sweeps, then restart from X0 so the timed sweeps are sweeps 1..K
    if args.warmup > 0:
        plan.run(args.warmup)
    plan.reset()
    _, s0 = plan.download()
    launches0 = plan.launches()
    sampler = ClockSampler(dev)
    barrier()
    sampler.start()
    plan.run(args.steps, sync=True)
    barrier()
    clocks = sampler.stop()
    ms_local = plan.last_run_ms()
    launches = plan.launches() - launches0
    _, s = plan.download()
    ms = max_over_ranks(ms_local)
    inter = (s.interactions_attr + s.interactions_rep) - (s0.interactions_attr + s0.interactions_rep)
    graph_launches = plan.graph_launches()
    sweeps = s.iterations_run
    # Per-phase device times come from events around every sweep's passes; the
    # timed run above replays sweeps 2.. as CUDA graphs (no per-sweep events), so
    # the same K sweeps run once more with every launch enqueued and that run
    # gives the fused kernel's own time (the roofline below), not the value.
    plan.set_graphs(False)
    plan.reset()
    barrier()
    plan.run(args.steps, sync=True)
    barrier()
    _, sp = plan.download()
    ms_nograph = max_over_ranks(plan.last_run_ms())
    kernel_ms = max_over_ranks(sp.kernel_ms)
    sort_ms = max_over_ranks(sp.sort_ms)
    plan.set_graphs(True)
    value = inter / (ms / 1e3)
    log(f"[rank {rank}] {args.steps} sweeps: {ms:.2f} ms, {value:.3e} interactions/s, "
        f"kernel {kernel_ms:.2f} ms, grid {sort_ms:.2f} ms, careful {s.careful_points}")

    # ---------------- roofline of the fused kernel ----------------
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    pk = sfu_peak(1965.0)
    # per-GPU rate of the dominant kernel: this GPU's share of the interactions over
    # the kernel's own device time (slowest rank)
    kernel_rate = (inter / world) / (kernel_ms / 1e3) if kernel_ms > 0 else 0.0
    roofline = {
        "bound": "sfu", "unit": "interactions/s",
        "achieved": kernel_rate,
        "peak": pk["peak"],
        "frac": kernel_rate / pk["peak"],
        "kernel": "fast_kernel attraction + repulsion passes (lop_fast.cu), per sweep",
        "kernel_share_of_step": kernel_ms / ms_nograph if ms_nograph > 0 else None,
        "peak_source": pk["source"] + " at sm_max 1965 MHz",
        "frac_at_measured_clock": kernel_rate / (pk["per_sm_clk"] * 148 * sm_mhz * 1e6),
        "traffic": None,
    }
    # the latest ncu --set full capture of the two passes (profiles/rNN_fast_kernel_ncu.json)
    cands = sorted(f for f in os.listdir(os.path.join(HERE, "profiles"))
                   if f.endswith("fast_kernel_ncu.json")) if os.path.isdir(os.path.join(HERE, "profiles")) else []
    prof = os.path.join(HERE, "profiles", cands[-1]) if cands else ""
    if prof and os.path.exists(prof):
        try:
            # DRAM bytes of one sweep's attraction + repulsion launches (ncu --set full)
            roofline["traffic"] = json.load(open(prof)).get("dram_bytes_per_launch")
            roofline["traffic_source"] = os.path.relpath(prof, HERE)
        except Exception:
            pass

    # ---------------- e2e through the public API ----------------
    e2e = None
    if not args.no_e2e:
        # steady state of a process that calls the API repeatedly: the device-side
        # plan of the timed region is released first (its memory returns to the
        # library's pool) and one untimed call warms the pinned staging buffers
        plan.close()
        prm2 = pb.LopParams(kernel=params.kernel, mu=params.mu, iterations=args.steps,
                            convergence_tol=params.convergence_tol)

        def e2e_call():
            if world == 1:
                return pb.lop_project(P, X0, prm2, eta=c["eta"], density_weights=c["wlop"],
                                      precision=precision, device=dev, lanes_per_point=args.lanes)
            p2 = make_plan()
            p2.upload(P, X0)
            p2.run(args.steps)
            res = p2.download()
            p2.close()
            return res

        e2e_call()
        barrier()
        t = time.perf_counter()
        out, se = e2e_call()
        wall = time.perf_counter() - t
        wall = max_over_ranks(wall)
        inter_e = se.interactions_attr + se.interactions_rep
        e2e = {"value": inter_e / wall, "unit": "interactions/s",
               "h2d_bytes_per_step": int((P.nbytes + X0.nbytes) / max(1, args.steps)),
               "d2h_bytes_per_step": int(out.nbytes / max(1, args.steps)),
               "h2d_bytes_total": int(P.nbytes + X0.nbytes), "d2h_bytes_total": int(out.nbytes),
               "wall_s": wall, "api": "pcs_lop_run (C ABI) with host buffers" if world == 1
               else "pcs_lop_plan_{create,set_comm,upload,run,download} with host buffers",
               "state": "warm process (second call; the library's device pool and pinned "
                        "staging buffers are reused, CUDA context already up)"}

    # ---------------- CPU baseline (rank 0, N = 1 only) ----------------
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu:
        Pb, Xb = P, X0
        if precision == "fp32":
            Pb = P.astype(np.float32).astype(np.float64)
            Xb = X0.astype(np.float32).astype(np.float64)
        try:
            cbr = cpu_baseline(cfg, Pb, Xb, c)
            cb = {k: cbr[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # pragma: no cover
            cb = {"value": None, "unit": "interactions/s", "cores": os.cpu_count(),
                  "kind": "unavailable", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "neighbour interactions/sec (LOP sweep)",
            "value": value, "unit": "interactions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / max(1, args.steps),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if precision == "fp32" else "f64",
            "data": "synthetic (seeded host generator, BASELINE.md §4)",
            "config": {"workload": WORKLOADS[cfg], "sweeps_timed": args.steps,
                       "sweeps_run": sweeps, "l2": "inputs larger than L2 (P = "
                       f"{P.shape[0] * 16 / 1e6:.0f} MB fp32 on device > 126 MB)",
                       "parallelism": f"dp{world}: P replicated, X sharded by cell-sorted ranges,"
                                      " NCCL all-gather of X per sweep" if world > 1 else "1 GPU"},
            "sweeps_per_s": args.steps / (ms / 1e3),
            "interactions_per_sweep": inter / max(1, args.steps),
            "kernel_ms_per_sweep": kernel_ms / max(1, args.steps),
            "grid_ms_per_sweep": sort_ms / max(1, args.steps),
            "careful_points": s.careful_points,
            "roofline": roofline,
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": launches,
            "cuda_graph_launches": graph_launches,
            "ms_per_step_without_graphs": ms_nograph / max(1, args.steps),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
