"""Developer tool: per-launch time / DRAM bytes / achieved GB/s from an ncu CSV
captured with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum."""
import csv
import sys
from collections import OrderedDict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
d = OrderedDict()
for r in rows:
    d.setdefault((r[ii], r[ki].split("(")[0].split("::")[-1]), {})[r[mi]] = \
        float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
print("| id | kernel | time (µs) | DRAM read (MB) | DRAM write (MB) | GB/s |")
print("|---:|---|---:|---:|---:|---:|")
for (i, k), m in d.items():
    t = m["gpu__time_duration.sum"]
    rb, wb = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    print(f"| {i} | {k} | {t * 1e6:.1f} | {rb / 1e6:.1f} | {wb / 1e6:.1f} | {(rb + wb) / t / 1e9:.0f} |")
