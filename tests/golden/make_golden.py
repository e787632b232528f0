#!/usr/bin/env python3
"""Generate the golden fixtures of tests/golden/ from the pinned CPU oracle.

The reference ships no stored vectors for the hot path; these are
produced by the oracle (oracle/ihs_oracle.cpp, libstdc++ 13.3 RNG types) in
this container and committed, so the GPU box can check the CUDA path against
fixed bytes even without rebuilding the oracle.

    python tests/golden/make_golden.py   # rewrites tests/golden/golden.npz
"""
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle import oracle as O  # noqa: E402


def main():
    out = {}
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
    np.savez_compressed(HERE / "golden.npz", **out)
    print("wrote", HERE / "golden.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
