#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X.csv):
per kernel name the launch count and mean time, then each step kernel's share of one step.

Usage: python tools/launch_summary.py launches.csv [--steps K] [--header "..."] [--out file.txt]
(K defaults to the launch count of k_norm_finalize, which runs once per step.)
The per-step share divides every lirank:: kernel's total by the launches it had per step
(launches // (warmup + steps) is not known here, so kernels launched exactly once per step
are the ones the bench's timed + warm-up steps run; setup kernels are listed but excluded)."""
import csv
import io
import sys
from collections import OrderedDict

SETUP = ("k_fill", "k_fill_table", "k_fill_grad", "k_flush", "k_quantize", "k_gather_rows_b",
         "k_scatter_rows_b")


def main():
    path = sys.argv[1]
    nsteps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 0
    header = sys.argv[sys.argv.index("--header") + 1] if "--header" in sys.argv else ""
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    out = []
    if header:
        out.append("# " + header)
    out.append("# Cold-cache serialised per-launch times (ncu replays each launch alone): compare SHARES of the")
    out.append("# step, not absolutes.")
    out.append(f"{'kernel':44s} {'launches':>8s} {'mean_us':>10s}")
    for k, (n, t) in agg.items():
        out.append(f"{k:44s} {n:8d} {t / n:10.1f}")
    if nsteps <= 0:  # a7's finalize runs exactly once per step
        nsteps = max([n for k, (n, _) in agg.items() if k.split("<")[0].endswith("k_norm_finalize")] or [1])
    step = OrderedDict()
    for k, (n, t) in agg.items():
        base = k.split("<")[0]
        if any(base.endswith(s) for s in SETUP):
            continue
        step[base] = step.get(base, 0.0) + t / nsteps
    tot = sum(step.values())
    out.append("")
    out.append(f"# share of one step (step kernels only; totals / {nsteps} steps)")
    for k, t in sorted(step.items(), key=lambda kv: -kv[1]):
        out.append(f"{k:44s} {t:10.1f} us {100 * t / tot:6.1f}%")
    out.append(f"{'total':44s} {tot:10.1f} us")
    text = "\n".join(out) + "\n"
    if "--out" in sys.argv:
        open(sys.argv[sys.argv.index("--out") + 1], "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
