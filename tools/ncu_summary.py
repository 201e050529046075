"""Summarise ncu evidence for profiles/ (run here, on the CPU side).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        [--rep gpurun_out/prof.ncu-rep] [--title ...] > profiles/rNN/summary.md

* launch list (``ncu --metrics gpu__time_duration.sum``): per-kernel launch
  count, total device time and share of the step;
* full capture (``ncu --set full``): per launch duration, DRAM bytes
  (traffic), FP64-pipe and issue utilisation, occupancy, registers.
"""
from __future__ import annotations

import argparse
import json
import collections
import csv
import io
import re
import subprocess

RAW = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "clk"),
]

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name: str) -> str:
    n = name
    for p in ("void ", "ppb::", "<unnamed>::", "(anonymous namespace)::"):
        n = n.replace(p, "")
    n = n.replace("unnamed>::", "")
    return n.split("(")[0].strip()


def launches(path: str):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= max(ki, vi, ui):
            continue
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-3)
        a = agg.setdefault(short(r[ki]), [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = ["| kernel | launches | total µs | avg µs | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(out)


def full(rep: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    cols = [(h.index(m), lbl, units[h.index(m)]) for m, lbl in RAW if m in h]
    ki = h.index("Kernel Name")
    out = ["| kernel | " + " | ".join(lbl for _, lbl, _ in cols) + " |",
           "|---" * (len(cols) + 1) + "|"]
    for r in rows[2:]:
        vals = []
        for i, lbl, u in cols:
            v = r[i]
            if lbl == "dur":
                v = f"{float(v) * SCALE.get(u, 1.0):.1f} µs"
            elif lbl.startswith("dram"):
                v = f"{float(v) * BYTES.get(u, 1) / 1e6:.2f} MB"
            vals.append(v)
        out.append(f"| `{short(r[ki])}` | " + " | ".join(vals) + " |")
    return "\n".join(out)


CATEGORY = [("band_run_kernel", "cost pass B (band tiles + candidate bins)"),
            ("band3_kernel", "cost pass B (band tiles + candidate bins)"),
            ("band_kernel", "cost pass B (band tiles + candidate bins)"),
            ("dp_pass_kernel<1", "DP bound pass (+ first candidate, fused)"),
            ("dp_pass_kernel<2", "DP bound pass (+ first candidate, fused)"),
            ("dp_pass_kernel<3", "DP bound pass (+ first candidate, fused)"),
            ("dp_pass_kernel<0", "DP candidate passes")]


def traffic(rep: str, plans: int, source: str) -> dict:
    """Per-plan DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of
    the bench's roofline kernels, averaged over the captured launches (the
    record bench.py reads as roofline.traffic)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    acc = {}
    for r in rows[2:]:
        cat = next((c for k, c in CATEGORY if short(r[ki]).startswith(k)), None)
        if cat is None:
            continue
        b = float(r[ri]) * BYTES.get(units[ri], 1) + float(r[wi]) * BYTES.get(units[wi], 1)
        n, t = acc.get(cat, (0, 0.0))
        acc[cat] = (n + 1, t + b)
    return {"source": source,
            "kernels": {c: {"dram_bytes_per_plan": t / n / plans, "launches_captured": n}
                        for c, (n, t) in acc.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--traffic", help="write the per-plan DRAM traffic record here (needs --rep)")
    ap.add_argument("--plans", type=int, default=148, help="mini-batches per captured launch")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    if a.traffic:
        with open(a.traffic, "w") as f:
            json.dump(traffic(a.rep, a.plans, a.source), f, indent=1)
    print(f"# {a.title}\n")
    if a.launches:
        print("## Launch list (`--metrics gpu__time_duration.sum --clock-control none`; cold, serialised)\n")
        print(launches(a.launches) + "\n")
    if a.rep:
        print("## Full capture (`--set full --clock-control none --import-source on`)\n")
        print(full(a.rep) + "\n")


if __name__ == "__main__":
    main()
