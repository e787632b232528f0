#!/usr/bin/env python3
"""Golden adaptive solves of the BASELINE configs at n/16 (tests/golden/configs_n16.npz).

SURVEY §8(d): parity for C3-C5 runs on down-scaled instances — the same seeded generator, d, nu and sigma,
n / 16 rows (n / 64 for the Gaussian C4) — where a single-thread CPU solve completes. Each case is solved here by the CPU oracle (pinned
bit-for-bit to the reference's own headers by tests/test_ref_pin.py; the configs' dense algebra makes a
reference-stub run of C4/C5 take hours) and the audit trail, counters and final iterate are committed; the GPU
test (tests/test_gpu_configs.py) regenerates the same data on the box (ihs.synth_generate, bit-exact with the
oracle's generator) and must reproduce the trail and counters exactly and x within 1e-10 in the Abar norm.

    python tests/golden/make_config_golden.py [case ...]   # ~30 min on 8 cores (cases run in parallel)
"""
import multiprocessing as mp
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

# (case, config, n, overrides of the bench knobs)
CASES = [
    ("c3_n16", "c3", 1 << 16, {}),
    ("c3_n16_default", "c3", 1 << 16, dict(m_initial=1, eps=1e-10)),
    ("c3_n16_norecompute", "c3", 1 << 16, dict(recompute_r_after_resketch=0)),
    ("c4_n16", "c4", 1 << 18, {}),
    # C4-Gaussian at n/64: the oracle's S*A at m = 8192 and n/16 would take hours single-threaded
    ("c4g_n64", "c4g", 1 << 16, dict(m_initial=4096, max_sketch=8192)),
    ("c5_n16", "c5", 62500, {}),
]


def solve_case(case):
    import bench
    from oracle import oracle as O
    name, cfg_name, n, over = case
    c = dict(bench.CONFIGS[cfg_name])
    d = c["d"]
    A, b, _ = O.synth(n, d, spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                      outlier_frac=c["outliers"], data_seed=0)
    knobs = dict(m_initial=c["m_initial"], eps=c["eps"], max_sketch=c["max_sketch"] or 0,
                 recompute_r_after_resketch=1)
    knobs.update(over)
    cfg = O.default_config(rho=c["rho"], sketch_kind=1 if c["sketch"] == "SRHT" else 0,
                           mode=1 if c["mode"] == "GradientOnly" else 0, seed=0,
                           enforce_validity=int(c["enforce_validity"]), **knobs)
    t0 = time.time()
    x, rep, log, _ = O.adaptive_solve(A, b, c["nu"], cfg, log_capacity=8192)
    xs = O.direct_solve(A, b, c["nu"])
    pe0 = O.prediction_error(A, b, c["nu"], np.zeros(d), xs)
    delta = np.sqrt(O.prediction_error(A, b, c["nu"], x, xs) / pe0)
    out = {
        f"{name}_spec": np.array([n, d], dtype=np.int64),
        f"{name}_knobs": np.array([knobs["m_initial"], knobs["max_sketch"], knobs["recompute_r_after_resketch"]],
                                  dtype=np.int64),
        f"{name}_eps": np.array([knobs["eps"]]),
        f"{name}_log": np.array([[e[0], e[1], e[4]] for e in log], dtype=np.int64),
        f"{name}_r": np.array([[e[2], e[3]] for e in log]),
        f"{name}_summary": np.array([rep.iterations, rep.rejections, rep.final_m, rep.converged,
                                     rep.sketch_exhausted], dtype=np.int64),
        f"{name}_counters": np.array([rep.counters.sketch, rep.counters.factor, rep.counters.solve,
                                      rep.counters.matvec], dtype=np.uint64),
        f"{name}_r1": np.array([rep.r1, rep.r_final]),
        f"{name}_x": x,
        f"{name}_delta": np.array([delta]),
    }
    print(f"{name}: T={rep.iterations} K={rep.rejections} m={rep.final_m} delta={delta:.2e} "
          f"{time.time() - t0:.0f}s", flush=True)
    return out


def main():
    want = sys.argv[1:]
    cases = [c for c in CASES if not want or c[0] in want]
    path = HERE / "configs_n16.npz"
    out = dict(np.load(path)) if path.exists() else {}
    with mp.Pool(len(cases)) as pool:
        for part in pool.imap_unordered(solve_case, cases):
            out.update(part)
    out["generator"] = np.array("oracle/ihs_oracle.cpp (pinned to the reference headers by tests/test_ref_pin.py)")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays")


if __name__ == "__main__":
    main()
