#!/usr/bin/env python3
"""Gradient-pass timing / profiling harness: python scripts/grad_bench.py [--n N] [--d D] [--reps R]
(one fused pass per call through the C-ABI, 1 right-hand side; synchronizes per call)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_05874_b200 import ihs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 19)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    A = np.empty((a.n, a.d), order="F")
    b = np.empty(a.n)
    ihs.synth_generate(a.n, a.d, spectrum=1, noise_std=0.01, data_seed=0, A_out=A, b_out=b)
    p = ihs.ProblemInstance(A, b, 1e-4)
    del A
    x = np.ones(a.d)
    for r in range(a.reps):
        t = time.perf_counter()
        ihs.gradient(p, x)
        print(f"grad n={a.n} d={a.d} wall_ms={1e3 * (time.perf_counter() - t):.3f}", flush=True)


if __name__ == "__main__":
    main()
