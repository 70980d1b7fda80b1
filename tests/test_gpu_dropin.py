"""Drop-in proof: the reference's own, unmodified proj/tests/test_lop.cpp runs
against this library (GPU).

tests/dropin/Makefile compiles /root/reference/proj/tests/test_lop.cpp with this
repo's include/pcs headers first on the include path and links
lib/libpcs_lop_b200.so.  The binary is built by __graft_entry__.build() where
the reference exists and travels with the repo snapshot to the GPU box.
"""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "dropin", "bin", "test_lop")


def test_reference_test_lop_passes_unmodified():
    if not os.path.exists(BIN):
        if os.path.isdir("/root/reference/proj/tests"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "dropin")], check=True)
        else:
            pytest.fail("tests/dropin/bin/test_lop was not built (run __graft_entry__.build() "
                        "where /root/reference exists)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "10 passed | 0 failed" in r.stdout
