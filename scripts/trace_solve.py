#!/usr/bin/env python3
"""Run a config's adaptive solve a few times with IHS_TRACE=1 (host timeline on stderr) and print the
device phase times of each: python scripts/trace_solve.py c3 [reps]"""
import json
import os
import sys

os.environ.setdefault("IHS_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2006_05874_b200 import ihs  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = bench.CONFIGS[name]
A = np.empty((c["n"], c["d"]), order="F")
b = np.empty(c["n"])
ihs.synth_generate(c["n"], c["d"], spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                   outlier_frac=c["outliers"], data_seed=0, A_out=A, b_out=b)
p = ihs.ProblemInstance(A, b, c["nu"])
cfg = bench.solver_config(ihs, c)
for i in range(reps):
    print(f"=== solve {i}", file=sys.stderr, flush=True)
    rep = ihs.adaptive_solve(p, cfg)
    print(json.dumps({"solve": i, **{k: v for k, v in rep.device_times.items()}}), flush=True)
