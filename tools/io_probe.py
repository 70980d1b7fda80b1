"""Developer probe: cloud IO of the config-3 data cloud (10M points, XYZ) —
B200 writer / reader (C ABI, host buffers in memory) vs the reference's
write_cloud_stream / read_cloud_stream (oracle/_ref; the reference's IO is
single-threaded)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2401_03365_b200 as pb  # noqa: E402
from oracle import oracle as O  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
P, _ = pb.generate_config(3, scale)
pb.format_cloud(P[:1000], device=0)  # context


def best(f, k=3):
    ts, r = [], None
    for _ in range(k):
        t = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t)
    return min(ts), r


tw, text = best(lambda: pb.format_cloud(P, "xyz", device=0))
tr, back = best(lambda: pb.parse_cloud(text, "xyz", device=0))
print(f"B200: {P.shape[0]} points, {len(text) / 1e6:.1f} MB: write {tw * 1e3:.1f} ms "
      f"({len(text) / tw / 1e9:.2f} GB/s), read {tr * 1e3:.1f} ms ({len(text) / tr / 1e9:.2f} GB/s)",
      flush=True)
if O.ref_available():
    t = time.perf_counter()
    rtext = O.ref_format_cloud(P, 0)
    rw = time.perf_counter() - t
    t = time.perf_counter()
    rback, err = O.ref_parse_cloud(rtext, 0)
    rr = time.perf_counter() - t
    same = rtext == text and err is None and np.array_equal(rback.view(np.uint64), back.view(np.uint64))
    print(f"reference: write {rw * 1e3:.0f} ms, read {rr * 1e3:.0f} ms; identical bytes and points: {same}",
          flush=True)
