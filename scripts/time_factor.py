"""SketchedSystem.factorize timing harness (host wall time per call, the call
synchronizes on the pivot check). Shapes: (m, d) pairs; k = d (Gram) when m >= d,
else k = m (Woodbury inner).

usage: python scripts/time_factor.py [--shapes 4096x256,1024x512,2048x1024,128x256] [--reps 20]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_05874_b200 import ihs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x256,1024x512,2048x1024,128x256")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    for sh in a.shapes.split(","):
        m, d = (int(v) for v in sh.split("x"))
        SA = np.asfortranarray(rng.standard_normal((m, d)))
        ihs.SketchedSystem.factorize(SA, 1e-3)  # warm
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            ihs.SketchedSystem.factorize(SA, 1e-3)
            ts.append(time.perf_counter() - t)
        print(f"factorize m={m} d={d} median_ms={1e3 * float(np.median(ts)):.3f} min_ms={1e3 * min(ts):.3f}", flush=True)


if __name__ == "__main__":
    main()
