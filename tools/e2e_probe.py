"""Developer probe: where the end-to-end (host-buffer) time of one run goes."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P, X0 = pb.generate_config(cfg)
prm, c = pb.config_params(cfg)
prm.iterations = 15
for rep in range(3):
    t0 = time.perf_counter()
    plan = pb.LopPlan(prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    t1 = time.perf_counter()
    plan.upload(P, X0)
    t2 = time.perf_counter()
    plan.run(15)
    t3 = time.perf_counter()
    dev_ms = plan.last_run_ms()
    out, s = plan.download()
    t4 = time.perf_counter()
    # the same download into pre-touched host buffers (no first-touch page faults)
    import ctypes as C
    from paper_2401_03365_b200 import _lib as L
    o2 = np.ones((plan.m, 3)); i2 = np.ones(max(plan.m, 1), dtype=np.uint32); sc = L.LopSummaryC()
    t6 = time.perf_counter()
    L.lib().pcs_lop_plan_download(plan._h, o2.ctypes.data_as(C.POINTER(C.c_double)), C.byref(sc),
                                  i2.ctypes.data_as(C.POINTER(C.c_uint32)), i2.size)
    t7 = time.perf_counter()
    print(f"download into touched buffers {1e3*(t7-t6):.1f} ms")
    plan.close()
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms upload {1e3*(t2-t1):.1f} ms (device setup {s.setup_ms:.1f}) "
          f"run {1e3*(t3-t2):.1f} ms (device {dev_ms:.1f}) "
          f"download {1e3*(t4-t3):.1f} ms close {1e3*(t5-t4):.1f} ms total {1e3*(t5-t0):.1f}")
    t0 = time.perf_counter()
    out, s = pb.lop_project(P, X0, prm, eta=c["eta"], density_weights=c["wlop"], precision="fp32")
    print(f"lop_project total {1e3*(time.perf_counter()-t0):.1f} ms setup {s.setup_ms:.1f} sweeps {s.sweeps_ms:.1f}")
