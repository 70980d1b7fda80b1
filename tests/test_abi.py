"""The C-ABI boundary (include/pcs_lop.h) on a CPU-only host.

No compute call reaches a device here: these tests check that the in-tree
library loads, exports every symbol the header declares, keeps the reference's
parameter defaults and validation order (proj/include/pcs/lop.hpp:12-35,
proj/src/lop.cpp:13-20), fails loudly without an sm_100 device, and that the
host generators reproduce the reference's draw order.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pcs_lop.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(pb):
    from paper_2401_03365_b200 import _lib
    lib = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTED)
    assert lib.pcs_lop_abi_version() == 1


def test_descriptor_defaults_match_reference(pb):
    from paper_2401_03365_b200 import _lib
    d = _lib.LopDesc()
    _lib.lib().pcs_lop_desc_default(C.byref(d))
    assert d.struct_size == C.sizeof(_lib.LopDesc)
    # KernelParams{h=1, cutoff=3} and LopParams{mu=0.4, iterations=30, tol=1e-7}
    assert (d.h, d.cutoff_multiple, d.mu, d.iterations, d.convergence_tol) == (1.0, 3.0, 0.4, 30, 1e-7)
    assert d.precision == _lib.PCS_PREC_FP64 and d.eta_kind == _lib.PCS_ETA_INV_CUBE
    assert d.density_weights == 0
    assert _lib.lib().pcs_lop_validate(C.byref(d)) == 0


@pytest.mark.parametrize("kw,msg", [
    (dict(h=0.0), "bandwidth"), (dict(h=-1.0), "bandwidth"), (dict(cutoff_multiple=0.0), "cutoff"),
    (dict(mu=0.5), "mu"), (dict(mu=-0.1), "mu"), (dict(iterations=0), "iterations"),
    (dict(convergence_tol=0.0), "convergence_tol"), (dict(eta_kind=7), "eta"),
    (dict(precision=3), "precision"), (dict(lanes_per_point=3), "lanes"),
])
def test_validation_errors(pb, kw, msg):
    from paper_2401_03365_b200 import _lib
    d = _lib.LopDesc()
    _lib.lib().pcs_lop_desc_default(C.byref(d))
    for k, v in kw.items():
        setattr(d, k, v)
    assert _lib.lib().pcs_lop_validate(C.byref(d)) == _lib.PCS_ERR_INVALID_PARAM
    assert msg in _lib.last_error()


def test_struct_size_guard(pb):
    from paper_2401_03365_b200 import _lib
    d = _lib.LopDesc()
    _lib.lib().pcs_lop_desc_default(C.byref(d))
    d.struct_size = 8
    assert _lib.lib().pcs_lop_validate(C.byref(d)) == _lib.PCS_ERR_INVALID_PARAM


def test_python_mirror_validation_order(pb):
    P = np.zeros((1, 3))
    # InvalidParam before EmptyCloud (lop.cpp:13-15), same as the reference test_lop.cpp:170-176
    with pytest.raises(pb.InvalidParam):
        pb.lop_project(np.zeros((0, 3)), P, pb.LopParams(kernel=pb.KernelParams(0.0)))
    with pytest.raises(pb.InvalidParam):
        pb.lop_project(P, P, pb.LopParams(mu=0.5))
    with pytest.raises(pb.InvalidParam):
        pb.lop_project(P, P, pb.LopParams(iterations=0))
    with pytest.raises(pb.EmptyCloud):
        pb.lop_project(np.zeros((0, 3)), P, pb.LopParams())
    # an empty initial set passes through without touching a device (lop.cpp:18-20)
    q, s = pb.lop_project(P, np.zeros((0, 3)), pb.LopParams())
    assert q.shape == (0, 3) and s.iterations_run == 0 and not s.converged


def test_no_cpu_fallback(pb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    P = np.random.default_rng(0).uniform(size=(10, 3))
    with pytest.raises(pb.DeviceUnavailable, match="no CPU fallback"):
        pb.lop_project(P, P[:3], pb.LopParams())
    with pytest.raises(pb.DeviceUnavailable):
        pb.radius_query_all(P, P, 0.1)


def test_generators_match_reference(pb, golden):
    for kind, name in enumerate(["plane", "sphere", "torus", "bump"]):
        assert np.array_equal(pb.generate_surface(name, 100, 7), golden[f"surface_{kind}"])
    assert np.array_equal(pb.add_noise(golden["noise_in"], 0.1, 9), golden["noise_out"])
    assert np.array_equal(pb.add_noise(np.zeros((1, 3)), 1.0, 1), golden["noise_kat"])


def test_config_generators(pb):
    sizes = {c: pb.config_sizes(c) for c in range(1, 6)}
    assert sizes == {1: (20000, 2000), 2: (1000000, 100000), 3: (10000000, 1000000),
                     4: (4000000, 400000), 5: (50000000, 5000000)}
    P, X0 = pb.generate_config(1)
    # X0 is a subset of P without replacement
    Pset = {tuple(p) for p in P}
    assert all(tuple(x) in Pset for x in X0) and len({tuple(x) for x in X0}) == len(X0)
    r = np.linalg.norm(P, axis=1)
    assert abs(r.mean() - 1.0) < 1e-3 and 0.005 < r.std() < 0.02   # unit sphere + sigma 0.01
    P3, X3 = pb.generate_config(3, 0.01)
    assert P3.shape == (100000, 3) and X3.shape == (10000, 3)
    assert np.all(np.abs(P3[:, :2]) <= 1.0)
    zres = P3[:, 2] - 0.1 * np.sin(8 * P3[:, 0]) * np.cos(8 * P3[:, 1])
    assert abs(zres.std() - 0.003) < 1e-4                             # noise on z only
    P2, _ = pb.generate_config(2, 0.02)
    assert P2.shape[0] == 19000 + 1000                                # 5% outliers appended
    P4, _ = pb.generate_config(4, 0.01)
    hist = np.histogram(P4[:, 2], bins=[-1.1, 0, 1.1])[0]
    assert hist[1] / hist[0] > 40                                     # e^{3.9 z} density
    P5, _ = pb.generate_config(5, 0.002)
    assert P5.shape == (100000, 3)
    # determinism
    assert np.array_equal(pb.generate_config(3, 0.001)[0], pb.generate_config(3, 0.001)[0])


def test_loopback_group_host_object(pb):
    """Loopback groups (in-process ranks) are host objects: creatable without a GPU,
    1..8 ranks, and a plan on a CPU-only host still fails loudly before using one."""
    from paper_2401_03365_b200 import _lib
    lib = _lib.lib()
    g = C.c_void_p()
    assert lib.pcs_loopback_group_create(2, C.byref(g)) == 0 and g.value
    lib.pcs_loopback_group_destroy(g)
    for bad in (0, 9):
        h = C.c_void_p()
        assert lib.pcs_loopback_group_create(bad, C.byref(h)) != 0
        assert b"1..8" in lib.pcs_last_error()
    assert lib.pcs_lop_plan_set_loopback(None, None, 0) != 0
