"""Summarise ncu captures for profiles/ (developer tool, runs where ncu is installed).

    python tools/ncu_summary.py full  REPORT.ncu-rep OUT.json   # one --set full capture
    python tools/ncu_summary.py launches LAUNCHES.csv OUT.md    # --metrics gpu__time_duration.sum list
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

FULL_KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__t_sector_hit_rate.pct",
    "smsp__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
    return v * scale if scale else None


def _one(h, u, v):
    res = {"kernel": v[h.index("Kernel Name")][:120]}
    for k in FULL_KEYS:
        if k in h:
            i = h.index(k)
            try:
                res[k] = {"value": float(v[i].replace(",", "")), "unit": u[i]}
            except ValueError:
                res[k] = {"value": v[i], "unit": u[i]}
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                val = float(v[i])
            except ValueError:
                continue
            if val >= 0.05:
                stalls[k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")] = round(val, 3)
    res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    rd = res.get("dram__bytes_read.sum")
    wr = res.get("dram__bytes_write.sum")
    if rd and wr:
        res["dram_bytes"] = to_bytes(rd["value"], rd["unit"]) + to_bytes(wr["value"], wr["unit"])
    return res


def full(rep, out):
    """Every kernel launch of the capture; dram_bytes_per_launch sums them (one sweep's
    attraction + repulsion passes when the capture holds that pair)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    kernels = [_one(h, u, v) for v in r[2:]]
    res = {"report": rep.split("/")[-1], "kernels": kernels}
    if all("dram_bytes" in k for k in kernels):
        res["dram_bytes_per_launch"] = sum(k["dram_bytes"] for k in kernels)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ik, im, iv, iu = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    t = collections.defaultdict(float)
    n = collections.Counter()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        us = float(r[iv].replace(",", "")) * scale[r[iu]]
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").split("<")[0].split("::")[-1]
        t[name] += us
        n[name] += 1
    tot = sum(t.values())
    lines = [f"Launch list `{path.split('/')[-1]}`: {sum(n.values())} launches, "
             f"{tot / 1e3:.2f} ms summed (ncu, serialised, cold caches).", "",
             "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {n[k]} | {v:.1f} | {v / tot * 100:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
