#!/usr/bin/env python3
"""Stopping-rule knob scan on the B200 at the BASELINE configs' full sizes.

For each config and each (m_initial, eps) pair, one adaptive_solve on the device and its true relative error
against the device direct_solve (problem.hpp:73-82):
  delta   = ||Abar (x - x*)|| / ||Abar x*||      (Abar = [A; nu I])
  pe_rel  = prediction_error(x) / prediction_error(0) = delta^2   (problem.hpp:104-109)
Used to choose the SolverConfig knobs under which "time to 1e-10" means a solve that reaches the target
(DESIGN.md §4). Usage: python scripts/knob_scan.py c3 "[1,1024,2048]" "[1e-10,1e-20]"
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("pathlib").Path(__file__).resolve().parents[1].as_posix())
import bench  # noqa: E402
from paper_2006_05874_b200 import ihs  # noqa: E402


def main():
    name = sys.argv[1]
    m_inits = eval(sys.argv[2])
    epss = eval(sys.argv[3])
    c = bench.CONFIGS[name]
    n, d, nu = c["n"], c["d"], c["nu"]
    A = np.empty((n, d), order="F")
    b = np.empty(n)
    ihs.synth_generate(n, d, spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                       outlier_frac=c["outliers"], data_seed=0, A_out=A, b_out=b)
    p = ihs.ProblemInstance(A, b, nu)
    del A
    t0 = time.time()
    xs = ihs.direct_solve(p)
    t_direct = time.time() - t0
    pe0 = ihs.prediction_error(p, np.zeros(d), xs)
    for mi in m_inits:
        for eps in epss:
            cfg = ihs.SolverConfig(rho=c["rho"], sketch_kind=getattr(ihs.SketchKind, c["sketch"]),
                                   mode=getattr(ihs.SolveMode, c["mode"]), m_initial=mi, eps=eps, seed=0)
            rep = ihs.adaptive_solve(p, cfg)  # warm (plans, pools)
            t0 = time.time()
            rep = ihs.adaptive_solve(p, cfg)
            wall = time.time() - t0
            pe = ihs.prediction_error(p, rep.x, xs)
            out = {"config": name, "m_initial": mi, "eps": eps, "T": rep.iterations, "K": rep.rejections,
                   "final_m": rep.final_m, "converged": rep.converged, "delta": float(np.sqrt(pe / pe0)),
                   "pe_rel": pe / pe0, "wall_s": wall, "direct_s": t_direct,
                   "m_schedule": [e.m for e in rep.log if int(e.branch) == 2],
                   "branches": "".join("PGR"[int(e.branch)] for e in rep.log)}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
