"""Sketch timing harness: one problem, a list of sketch sizes, wall time per
call (includes the host-side sampling and the SA read-back). Meant to run under
`ncu --metrics gpu__time_duration.sum` for per-kernel device times; it exits 0
whatever the numerics (timing experiments may use wrong-result debug modes).

usage: python scripts/time_sketch.py [--n N] [--d D] [--kind srht|gaussian] [--ms 2,64,2048] [--reps R]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2006_05874_b200 import ihs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--kind", default="srht", choices=["srht", "gaussian"])
    ap.add_argument("--ms", default="2,64,512,2048")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    A, b, _ = ihs.synth_generate(a.n, a.d, decay=0.99)
    P = ihs.ProblemInstance(A, b, 1e-3)
    del A
    fn = ihs.srht_sketch if a.kind == "srht" else ihs.gaussian_sketch
    for m in [int(x) for x in a.ms.split(",")]:
        for r in range(a.reps):
            t = time.perf_counter()
            fn(P, m, 12345 + r)
            print(f"{a.kind} m={m} rep={r} wall_ms={1e3 * (time.perf_counter() - t):.3f}", flush=True)


if __name__ == "__main__":
    main()
