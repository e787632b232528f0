#!/usr/bin/env python3
"""Device sketch timing at a config's shape (no SA read-back): wall time of ihs_gpu_sketch with SA_out = NULL
(the call ends with a stream synchronize, so this is device time + the host's row sampling / tile planning).

usage: python scripts/sketch_bench.py [--config c4] [--kind srht|gaussian] [--ms 8192,32768,131072] [--reps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2006_05874_b200 import ihs  # noqa: E402
from paper_2006_05874_b200._lib import lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--kind", default="srht", choices=["srht", "gaussian"])
    ap.add_argument("--ms", default="8192,32768,131072")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--d", type=int, default=0, help="override the column count (profiling at the config's n)")
    a = ap.parse_args()
    c = dict(bench.CONFIGS[a.config])
    if a.d:
        c["d"] = a.d
    A = np.empty((c["n"], c["d"]), order="F")
    b = np.empty(c["n"])
    ihs.synth_generate(c["n"], c["d"], spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                       outlier_frac=c["outliers"], data_seed=0, A_out=A, b_out=b)
    P = ihs.ProblemInstance(A, b, c["nu"])
    del A
    kind = 1 if a.kind == "srht" else 0
    n_pad = 1 << (c["n"] - 1).bit_length()
    for m in [int(x) for x in a.ms.split(",")]:
        ts = []
        for r in range(a.reps + 1):
            t = time.perf_counter()
            st = lib().ihs_gpu_sketch(P.handle, kind, m, 12345 + r, None, None)
            assert st == 0, lib().ihs_gpu_last_error()
            ts.append(1e3 * (time.perf_counter() - t))
        ms = float(np.median(ts[1:]))
        algo = 8.0 * c["n"] * c["d"] + 8.0 * m * c["d"]
        print(f"{a.config} {a.kind} m={m} ms={ms:.3f} algo_GBps={algo / ms / 1e6:.0f} all={[round(x, 2) for x in ts]}",
              flush=True)


if __name__ == "__main__":
    main()
