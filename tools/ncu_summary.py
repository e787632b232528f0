#!/usr/bin/env python3
"""Summarize an ncu --csv launch list (gpu__time_duration.sum per launch):
per-kernel count, total and mean device time, and share of the total.

    python tools/ncu_summary.py gpurun_out/launches_c2.csv [--skip-first N]
"""
import collections
import csv
import io
import re
import sys


def load(path):
    text = open(path, errors="replace").read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        name = re.sub(r"^void ", "", name)
        out.append((int(r["ID"]), name, v * scale))
    return out


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip-first") + 1]) if "--skip-first" in sys.argv else 0
    rows = load(path)[skip:]
    agg = collections.OrderedDict()
    for _, name, ms in rows:
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ms)
    total = sum(t for _, t in agg.values())
    print(f"{len(rows)} launches, {total:.3f} ms total (serialised, cold cache)")
    print(f"{'kernel':60s} {'count':>6s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
    for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {c:6d} {t:10.3f} {1e3 * t / c:10.2f} {100 * t / total:6.1f}%")


if __name__ == "__main__":
    main()
