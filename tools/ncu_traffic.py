#!/usr/bin/env python3
"""Summarise an `ncu --set full` capture (.ncu-rep) into profiles/.

    python tools/ncu_traffic.py REPORT.ncu-rep CFG OUT.txt [--role REGEX=ROLE ...]

Writes a per-launch table (duration, DRAM read/write bytes, DRAM and SM
throughput, achieved occupancy, registers, top warp-stall reasons) to OUT.txt
and records the DRAM bytes per launch of each role (e.g. "sketch", "gradient")
in profiles/traffic.json, which bench.py reports as roofline.traffic. When
several launches map to one role, the last captured launch of each kernel
name is used and the names are summed (an SRHT sketch = phase 1 + phase 2).
"""
import csv
import io
import json
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def val(d, u, k):
    v = d.get(k, "")
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * UNIT.get(u.get(k, ""), 1.0)


def main():
    report, cfg, out_txt = sys.argv[1:4]
    roles = [a.split("=", 1) for a in sys.argv[4:] if "=" in a]
    launches = raw(report)
    lines = [f"ncu --set full summary of {pathlib.Path(report).name} ({cfg}); bytes are per launch", ""]
    stall_keys = None
    per_role = {}
    for d, u in launches:
        name = re.sub(r"\(.*", "", d.get("Kernel Name", "?")).replace("void ", "")
        ms = val(d, u, "gpu__time_duration.sum")
        rd, wr = val(d, u, "dram__bytes_read.sum") or 0.0, val(d, u, "dram__bytes_write.sum") or 0.0
        if stall_keys is None:
            stall_keys = [k for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
                          not k.endswith("_not_issued")]
        stalls = sorted(((val(d, u, k) or 0.0, k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for k in stall_keys), reverse=True)
        tot = sum(s for s, _ in stalls) or 1.0
        top = ", ".join(f"{k} {100 * s / tot:.0f}%" for s, k in stalls[:4])
        gbs = (rd + wr) / (ms * 1e-3) / 1e9 if ms else 0.0
        lines.append(f"{name}")
        lines.append(f"  grid {d.get('launch__grid_size')} x {d.get('launch__block_size')}, "
                     f"{d.get('launch__registers_per_thread')} regs, duration {ms:.4f} ms")
        lines.append(f"  DRAM read {rd / 1e9:.4f} GB  write {wr / 1e9:.4f} GB  -> {gbs:.0f} GB/s "
                     f"(dram {d.get('dram__throughput.avg.pct_of_peak_sustained_elapsed')}% of peak, "
                     f"SM {d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')}%, "
                     f"warps active {d.get('sm__warps_active.avg.pct_of_peak_sustained_active')}%)")
        lines.append(f"  top stalls: {top}")
        for rx, role in roles:
            if re.search(rx, name):
                per_role.setdefault(role, {})[name] = rd + wr
    pathlib.Path(out_txt).write_text("\n".join(lines) + "\n")
    tj = ROOT / "profiles" / "traffic.json"
    data = json.loads(tj.read_text()) if tj.exists() else {}
    for role, by_name in per_role.items():
        data.setdefault(cfg, {})[role] = sum(by_name.values())
    tj.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print("\n".join(lines))
    print("traffic.json:", json.dumps(data.get(cfg, {})))


if __name__ == "__main__":
    main()
