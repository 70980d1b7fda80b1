"""Generates tests/golden/reference_io.npz from the UNMODIFIED reference's cloud
IO (pcs::write_cloud_stream / read_cloud_stream, proj/src/io.cpp, compiled into
oracle/_ref):

    python tests/golden/make_golden_io.py

Stored: a seeded cloud with special values, the reference's XYZ and PLY bytes
for it, and for a set of malformed / unusual texts either the parsed points or
the ParseError (line, message).  Pins the B200 writer and reader where
/root/reference does not exist (tests/test_gpu_io.py).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
from test_gpu_io import PLY_CASES, XYZ_CASES, special_cloud  # noqa: E402


def main():
    O.build(reference=True)
    assert O.ref_available()
    out = {}
    X = special_cloud(np.random.default_rng(31))
    out["cloud"] = X
    out["cloud_xyz"] = np.frombuffer(O.ref_format_cloud(X, 0), np.uint8)
    out["cloud_ply"] = np.frombuffer(O.ref_format_cloud(X, 1), np.uint8)
    for fmt, cases in ((0, XYZ_CASES), (1, PLY_CASES)):
        for name, text in cases.items():
            key = f"case_{fmt}_{name}"
            out[key + "_text"] = np.frombuffer(text, np.uint8)
            pts, err = O.ref_parse_cloud(text, fmt)
            if err is None:
                out[key + "_points"] = pts
            else:
                out[key + "_line"] = np.array(err[0])
                out[key + "_msg"] = np.frombuffer(err[1].encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "reference_io.npz"), **out)
    print("wrote reference_io.npz with", len(out), "arrays")


if __name__ == "__main__":
    main()
