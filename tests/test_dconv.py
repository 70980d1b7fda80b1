"""The double<->text conversions of the cloud IO kernels (csrc/dconv.h: Ryu
shortest formatting, exact-integer parsing) checked on the host against
libstdc++'s std::to_chars / std::from_chars — the functions the reference's
writer and reader call (proj/src/io.cpp:36-48, :240-245): every random bit
pattern, coordinate-like value and decimal string must format byte-identically
and parse bit-identically (or be left to the host parser)."""
import os
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("dconv") / "dconv_test")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I",
                    os.path.join(ROOT, "paper_2401_03365_b200", "csrc"),
                    os.path.join(ROOT, "tests", "dconv_host_test.cpp"), "-o", out], check=True)
    return out


@pytest.mark.parametrize("seed", [1, 2])
def test_format_and_parse_match_libstdcxx(binary, seed):
    r = subprocess.run([binary, "400000", str(seed)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "format: 0 mismatches" in r.stdout
    assert "parse: 0 mismatches" in r.stdout
