#!/usr/bin/env python3
"""Smoke-sized cases of the hot kernels for compute-sanitizer (memcheck / racecheck / synccheck):
SRHT (TMA phase 1 + three-round and two-round emitting passes, compact T), Gaussian sketch (MT19937 substreams,
polar acceptance, DMMA GEMM), the fused gradient (bulk-TMA panels, mbarrier ring, named barriers, PDL chain),
the sketched-system factorization (SYRK, blocked Cholesky, triangular inverse, W^T W) and one adaptive solve.

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_05874_b200 import ihs  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    # SRHT: n_pad = 2^13 (two-round pass), 2^21 (three-round pass over a few columns), 2^20 compact T
    for n, d, m in ((5000, 4, 300), ((1 << 20) + 7, 2, 3000), ((1 << 20) - 3, 2, 50)):
        A = np.asfortranarray(rng.standard_normal((n, d)))
        ihs.srht_sketch(A, m, 1)
    A, b, _ = ihs.synth_generate(8192, 96, decay=0.95, noise_std=0.01, data_seed=1)
    ihs.gaussian_sketch(A, 256, 2)
    p = ihs.ProblemInstance(A, b, 1e-2)
    ihs.gradient(p, np.ones(96))
    SA = np.asfortranarray(rng.standard_normal((600, 96)))
    sys_ = ihs.SketchedSystem.factorize(SA, 0.5)
    sys_.solve(np.ones(96))
    SAw = np.asfortranarray(rng.standard_normal((40, 96)))  # Woodbury branch
    ihs.SketchedSystem.factorize(SAw, 0.5).solve(np.ones(96))
    rep = ihs.adaptive_solve(p, ihs.SolverConfig(sketch_kind=ihs.SketchKind.SRHT, m_initial=192, eps=1e-14))
    assert rep.converged
    print("sanitize case done", rep.iterations, rep.final_m)


if __name__ == "__main__":
    main()
