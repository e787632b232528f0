#!/usr/bin/env python3
"""Generate the golden fixtures of tests/golden/ from the REFERENCE ITSELF.

The reference ships no stored vectors for the hot path. These are
produced in this container by oracle/_ref/libihs_ref.so — the reference's own
headers (/root/reference/proj/include/ihs/*.hpp) compiled unchanged against
the Eigen-API subset in oracle/eigen_stub (`make -C oracle ref`, libstdc++ 13.3
RNG types) — and committed, so the GPU box (where /root/reference does not
exist) checks the CUDA path and the oracle restatement against the reference's
bytes. tests/test_golden.py holds the oracle to them as well.

    make -C oracle ref && python tests/golden/make_golden.py   # rewrites tests/golden/golden.npz
"""
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle import ref as O  # noqa: E402  (the reference code; same signatures as oracle/oracle.py)


def main():
    if not O.AVAILABLE:
        raise SystemExit("oracle/_ref/libihs_ref.so missing: run `make -C oracle ref` (needs /root/reference)")
    out = {"generator": np.array("oracle/_ref: reference headers proj/include/ihs/*.hpp + oracle/eigen_stub")}
    # raw streams and the derived D / P of a few sub-seeds (rng.hpp:30-66)
    for i, (seed, K) in enumerate([(0, 0), (0, 5), (12345, 11)]):
        sub = O.derive_seed(seed, K)
        out[f"derive_{i}"] = np.array([seed, K, sub], dtype=np.uint64)
        out[f"mt_raw_{i}"] = O.mt_raw(O.derive_seed(sub, 1), 1024)
        out[f"signs_{i}"] = O.rademacher(O.derive_seed(sub, 1), 4096).astype(np.int8)
        out[f"rows_{i}"] = O.sample_without_replacement(O.derive_seed(sub, 2), 4096, 257)
        out[f"normals_{i}"] = O.fill_gaussian(O.derive_seed(sub, 0), 37, 29, 1.0 / np.sqrt(37.0))
    # SRHT / Gaussian sketches of a fixed synthetic matrix (sketch.hpp:58-108)
    A, b, xt = O.synth(3000, 12, decay=0.9, noise_std=0.01, outlier_frac=0.01, data_seed=7)
    out["A"] = A
    out["b"] = b
    for m, seed in [(1, 0), (64, 3), (4096, 9)]:
        out[f"srht_m{m}_s{seed}"] = O.srht_sketch(A, m, seed)
    out["gauss_m40_s2"] = O.gaussian_sketch(A, 40, 2)
    # one adaptive solve per sketch kind: audit trail and final iterate (solver.hpp:106-232)
    for kind, name in [(0, "gauss"), (1, "srht")]:
        x, rep, log, _ = O.adaptive_solve(A, b, 0.05, O.default_config(sketch_kind=kind, seed=3))
        out[f"solve_{name}_x"] = x
        out[f"solve_{name}_log"] = np.array([[l[0], l[1], l[4]] for l in log], dtype=np.int64)
        out[f"solve_{name}_summary"] = np.array([rep.iterations, rep.rejections, rep.final_m, rep.converged],
                                                dtype=np.int64)
        out[f"solve_{name}_counters"] = np.array([rep.counters.sketch, rep.counters.factor, rep.counters.solve,
                                                  rep.counters.matvec], dtype=np.uint64)
    # the CG / PCG comparators (baselines.hpp) and the exact minimizer on the same data
    for kind, name in [(0, "gauss"), (1, "srht")]:
        x, res, rep = O.pcg_solve(A, b, 0.05, kind, 4, 0.5, 1e-10, 100)
        out[f"pcg_{name}_x"] = x
        out[f"pcg_{name}_res"] = res
        out[f"pcg_{name}_summary"] = np.array([rep.iterations, rep.m, rep.converged, rep.setup_flops], dtype=np.int64)
    x, res, rep = O.cg_solve(A, b, 0.05, 1e-8, 200)
    out["cg_x"], out["cg_res"] = x, res
    out["cg_summary"] = np.array([rep.iterations, rep.converged], dtype=np.int64)
    out["direct_x"] = O.direct_solve(A, b, 0.05)
    # the dual solver (dual.hpp) on an underdetermined instance (40 x 300)
    Au, bu, _ = O.synth(300, 40, decay=0.95, noise_std=0.01, data_seed=8)
    Au = np.asfortranarray(Au.T)
    bu = bu[:40].copy()
    out["Au"], out["bu"] = Au, bu
    x, z, rep, log, _ = O.solve_underdetermined(Au, bu, 0.3, O.default_config(seed=5))
    out["dual_x"], out["dual_z"] = x, z
    out["dual_summary"] = np.array([rep.iterations, rep.rejections, rep.final_m, rep.converged], dtype=np.int64)
    np.savez_compressed(HERE / "golden.npz", **out)
    print("wrote", HERE / "golden.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
