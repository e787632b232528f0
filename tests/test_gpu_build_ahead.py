"""Doublings built ahead (runtime.cpp, adaptive_solve_impl): on small problems the adaptive loop sketches and
factors doublings K+1 .. K+depth on side streams while it evaluates candidates under system K, and adopts them
in order. The sketch sequence is fixed in advance (solver.hpp:210-213: doubling K is m_initial 2^K rows with
derive_seed(seed, K)), so the result must not depend on it. Its systems also replay their factorization chains
as CUDA graphs (system_factorize; captured the second time a shape recurs, so the third solve of a problem
replays). The same solves with IHS_SPEC_DEPTH = 0 and IHS_FACTOR_GRAPH = 0 (everything on the solve stream as
plain launches, the reference's order) and with depths 1, 3 and 8 (graphs on) must give bit-identical iterates,
the same audit trail and the same cost counters — including solves that stop before adopting every built doubling (the
unadopted builds are charged nothing), Gaussian sketches, recompute_r_after_resketch = false, the Woodbury-to-Gram
switch (m crossing d) and repeated solves of one problem (the pool of systems is reused).

The depth is read once per process, so each depth runs in its own interpreter.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2006_05874_b200 import ihs
cases = json.loads(sys.argv[2])
out = []
for cs in cases:
    A, b, _ = ihs.synth_generate(cs["n"], cs["d"], spectrum=0, decay=0.95, noise_std=0.1, outlier_frac=0.0,
                                 data_seed=cs["seed"])
    p = ihs.ProblemInstance(A, b, cs["nu"])
    for rep_i in range(cs.get("reps", 1)):
        cfg = ihs.SolverConfig(sketch_kind=getattr(ihs.SketchKind, cs["kind"]), m_initial=cs["m0"], eps=cs["eps"],
                               seed=cs["seed"], rho=cs.get("rho", 0.1),
                               recompute_r_after_resketch=cs.get("recompute", True),
                               max_sketch=cs.get("max_sketch", 0) or None)
        r = ihs.adaptive_solve(p, cfg)
        c = r.counters
        out.append({"x": np.asarray(r.x).tobytes().hex(), "log": [(e.t, e.m, int(e.branch)) for e in r.log],
                    "sum": [r.iterations, r.rejections, r.final_m, int(r.converged)],
                    "cnt": [c.sketch, c.factor, c.solve, c.matvec]})
print(json.dumps(out))
"""

CASES = [
    dict(n=8192, d=256, nu=1e-3, kind="SRHT", m0=1, eps=1e-27, seed=0, reps=3),    # C1's shape and knobs
    dict(n=4096, d=96, nu=1e-2, kind="SRHT", m0=1, eps=1e-10, seed=3),             # stops with builds unadopted
    dict(n=3000, d=64, nu=1e-2, kind="Gaussian", m0=2, eps=1e-14, seed=5, reps=3),
    dict(n=5000, d=128, nu=1e-2, kind="SRHT", m0=4, eps=1e-16, seed=7, recompute=False),
    dict(n=2048, d=200, nu=1e-1, kind="SRHT", m0=1, eps=1e-20, seed=11, max_sketch=512),
]


def _run(depth, graph=True):
    env = dict(os.environ, IHS_SPEC_DEPTH=str(depth), IHS_FACTOR_GRAPH="1" if graph else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, json.dumps(CASES)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_build_ahead_is_bit_identical_to_in_order_solves():
    base = _run(0, graph=False)
    assert any(len([e for e in o["log"] if e[2] == 2]) >= 5 for o in base)  # the cases do resketch
    for depth in (1, 3, 8):
        got = _run(depth)
        assert len(got) == len(base)
        for i, (g, b) in enumerate(zip(got, base)):
            assert g["log"] == b["log"], (depth, i)
            assert g["sum"] == b["sum"], (depth, i)
            assert g["cnt"] == b["cnt"], (depth, i)
            assert g["x"] == b["x"], (depth, i)
    xs = [np.frombuffer(bytes.fromhex(o["x"]), dtype=np.float64) for o in base]
    assert all(np.all(np.isfinite(x)) and np.linalg.norm(x) > 0 for x in xs)
