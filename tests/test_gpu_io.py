"""Parity of the B200 cloud IO (csrc/io.cu) with the reference's
write_cloud_stream / read_cloud_stream (proj/src/io.cpp), run live through
oracle/_ref: identical bytes from the writer, bit-identical points from the
reader, and for malformed input the same ParseError line and message."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FMT = {"xyz": 0, "ply": 1}


@pytest.fixture(scope="module")
def ref(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not present")
    return orc


def special_cloud(rng):
    v = np.array([0.0, -0.0, 1.0, -1.0, 0.1, 1e22, 1e23, 5e-324, 2.2250738585072014e-308,
                  1.7976931348623157e308, 9007199254740993.0, 1.2345678901234568e20,
                  123456789012345678.0, 1e-5, 1.5e-5, 1e15, 1e16, 1e21, 12345678901234567890.0,
                  1.25e-6, 1e100, 4.35e17, 1 / 3, -2 / 3, 1e-300, 123456.0])
    bits = rng.integers(0, 2**63, 3000, dtype=np.int64).view(np.float64)
    bits = bits[np.isfinite(bits)]
    coords = rng.uniform(-2, 2, 3000) * 10.0 ** rng.integers(-4, 5, 3000)
    allv = np.concatenate([v, bits, coords, -coords[:500]])
    allv = allv[: len(allv) // 3 * 3]
    return allv.reshape(-1, 3)


@pytest.mark.parametrize("fmt", ["xyz", "ply"])
def test_writer_bytes_identical(pb, ref, fmt):
    rng = np.random.default_rng(21)
    for X in (special_cloud(rng), rng.normal(size=(5000, 3)), np.zeros((0, 3))):
        assert pb.format_cloud(X, fmt, device=0) == ref.ref_format_cloud(X, FMT[fmt])


@pytest.mark.parametrize("fmt", ["xyz", "ply"])
def test_reader_bit_exact_and_round_trip(pb, ref, fmt):
    rng = np.random.default_rng(22)
    X = special_cloud(rng)
    text = ref.ref_format_cloud(X, FMT[fmt])
    got = pb.parse_cloud(text, fmt, device=0)
    want, err = ref.ref_parse_cloud(text, FMT[fmt])
    assert err is None
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(got.view(np.uint64), X.view(np.uint64))  # shortest form round-trips
    assert pb.format_cloud(got, fmt, device=0) == text              # byte-stable


XYZ_CASES = {
    "comments_blank_crlf_tabs": b"# header\r\n\r\n  1 2 3\r\n\t4\t5\t6 \n   # indented comment\n7 8 9",
    "hard_numbers": b"1.2345678901234567890123 1e-300 3\n12345678901234567890 1e40 -0.0000000000000000000000000000001\n",
    "vertical_tab_blank": b"1 2 3\n\x0b\x0c \n4 5 6\n",
    "bad_count": b"0 0 0\n1 2\n",
    "too_many": b"1 2 3 4\n",
    "not_a_number": b"1 2 x\n",
    "nan": b"0 0 nan\n",
    "inf": b"inf 0 0\n",
    "out_of_range": b"0 0 1e999\n",
    "plus_sign": b"+1 2 3\n",
    "second_of_two_errors": b"1 2 3\n4 5 six\n7 8\n",
    "empty": b"",
}


@pytest.mark.parametrize("case", sorted(XYZ_CASES))
def test_xyz_reader_cases_match_reference(pb, ref, case):
    text = XYZ_CASES[case]
    want, err = ref.ref_parse_cloud(text, 0)
    if err is None:
        got = pb.parse_cloud(text, "xyz", device=0)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    else:
        with pytest.raises(pb.ParseError) as e:
            pb.parse_cloud(text, "xyz", device=0)
        assert (e.value.line, str(e.value)) == err


PLY_CASES = {
    "minimal": b"ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\nproperty float y\nproperty float z\nend_header\n1 2 3\n4 5 6\n",
    "extra_props_positional": b"ply\nformat ascii 1.0\ncomment c\nelement vertex 2\nproperty float nx\nproperty float z\nproperty float y\nproperty float x\nend_header\n9 1 2 3\n9 4 5 6\n",
    "faces_after": b"ply\nformat ascii 1.0\nelement vertex 3\nproperty double x\nproperty double y\nproperty double z\nelement face 1\nproperty list uchar int vertex_indices\nend_header\n0 0 0\n1 0 0\n\n0 1 0\n3 0 1 2\n",
    "other_element_first": b"ply\nformat ascii 1.0\nelement edge 1\nproperty int a\nelement vertex 1\nproperty double x\nproperty double y\nproperty double z\nend_header\n7\n1.5 2.5 3.5\n",
    "short_file": b"ply\nformat ascii 1.0\nelement vertex 3\nproperty double x\nproperty double y\nproperty double z\nend_header\n1 2 3\n",
    "bad_value": b"ply\nformat ascii 1.0\nelement vertex 2\nproperty double x\nproperty double y\nproperty double z\nend_header\n1 2 3\n1 2 q\n",
    "wrong_count": b"ply\nformat ascii 1.0\nelement vertex 1\nproperty double x\nproperty double y\nproperty double z\nend_header\n1 2\n",
    "binary": b"ply\nformat binary_little_endian 1.0\nend_header\n",
    "no_vertex": b"ply\nformat ascii 1.0\nelement face 0\nproperty list uchar int vertex_indices\nend_header\n",
    "missing_z": b"ply\nformat ascii 1.0\nelement vertex 1\nproperty double x\nproperty double y\nend_header\n1 2\n",
    "no_magic": b"plx\n",
}


@pytest.mark.parametrize("case", sorted(PLY_CASES))
def test_ply_reader_cases_match_reference(pb, ref, case):
    text = PLY_CASES[case]
    want, err = ref.ref_parse_cloud(text, 1)
    if err is None:
        got = pb.parse_cloud(text, "ply", device=0)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    else:
        with pytest.raises(pb.ParseError) as e:
            pb.parse_cloud(text, "ply", device=0)
        assert (e.value.line, str(e.value)) == err


def test_config3_scale_write_read(pb, ref):
    """3M points of the config-3 data cloud (30% scale): writer bytes equal the
    reference's, the reader returns the exact doubles."""
    P, _ = pb.generate_config(3, 0.3)
    text = pb.format_cloud(P, "xyz", device=0)
    assert text == ref.ref_format_cloud(P, 0)
    back = pb.parse_cloud(text, "xyz", device=0)
    assert np.array_equal(back.view(np.uint64), P.view(np.uint64))


def test_mesh_and_format_double(pb, ref):
    quad = (b"ply\nformat ascii 1.0\nelement vertex 4\nproperty double x\nproperty double y\n"
            b"property double z\nelement face 1\nproperty list uchar int vertex_indices\n"
            b"end_header\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n4 0 1 2 3\n")
    T = pb.parse_mesh(quad)
    assert T.shape == (2, 3, 3)
    assert np.array_equal(T[1], [[0, 0, 0], [1, 1, 0], [0, 1, 0]])
    with pytest.raises(pb.ParseError):
        pb.parse_mesh(quad.replace(b"4 0 1 2 3", b"4 0 1 2 9"))
    for v in (0.1, 1e22, 5e-324, -0.0, 123456789012345678.0):
        assert pb.format_double(v) == ref.ref_format_cloud(np.array([[v, 0, 0]]), 0).split(b" ")[0].decode()


def test_against_reference_fixture(pb):
    """The same checks against tests/golden/reference_io.npz (made by the
    reference, tests/golden/make_golden_io.py) — no reference build needed."""
    import os
    from conftest import ROOT
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_io.npz"))
    X = g["cloud"]
    assert pb.format_cloud(X, "xyz", device=0) == g["cloud_xyz"].tobytes()
    assert pb.format_cloud(X, "ply", device=0) == g["cloud_ply"].tobytes()
    for key in g.files:
        if not key.endswith("_text"):
            continue
        base = key[: -len("_text")]
        fmt = "xyz" if base.startswith("case_0_") else "ply"
        text = g[key].tobytes()
        if base + "_points" in g.files:
            got = pb.parse_cloud(text, fmt, device=0)
            assert np.array_equal(got.view(np.uint64), g[base + "_points"].view(np.uint64)), base
        else:
            with pytest.raises(pb.ParseError) as e:
                pb.parse_cloud(text, fmt, device=0)
            assert e.value.line == int(g[base + "_line"]), base
            assert str(e.value) == g[base + "_msg"].tobytes().decode(), base


def test_write_cloud_file_equals_format_cloud(pb, tmp_path):
    """write_cloud (caller-side buffer, no intermediate bytes) writes exactly the
    bytes format_cloud returns, in both formats, and read_cloud restores the
    points bit for bit; empty clouds included."""
    rng = np.random.default_rng(5)
    X = rng.normal(size=(5000, 3)) * np.array([1.0, 1e-9, 1e12])
    for fmt in ("xyz", "ply"):
        for cloud in (X, X[:0]):
            path = str(tmp_path / f"c{len(cloud)}.{fmt}")
            pb.write_cloud(cloud, path, device=0)
            data = open(path, "rb").read()
            assert data == pb.format_cloud(cloud, fmt, device=0)
            back = pb.read_cloud(path, device=0)
            assert np.array_equal(back.view(np.uint64), np.ascontiguousarray(cloud).view(np.uint64))
