#!/usr/bin/env python3
"""Host + device timeline (IHS_TRACE=1, stderr) of upload_async + adaptive_solve at a config's shape, and the wall
time of each round: python scripts/e2e_trace.py c3 [reps]"""
import os
import sys
import time

os.environ.setdefault("IHS_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402,F401
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2006_05874_b200 import ihs  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = bench.CONFIGS[name]
A_t = torch.empty((c["d"], c["n"]), dtype=torch.float64, pin_memory=True)
b_t = torch.empty((c["n"],), dtype=torch.float64, pin_memory=True)
A, b = A_t.numpy().T, b_t.numpy()
ihs.synth_generate(c["n"], c["d"], spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                   outlier_frac=c["outliers"], data_seed=0, A_out=A, b_out=b)
p = ihs.ProblemInstance(A, b, c["nu"])
cfg = bench.solver_config(ihs, c)
ihs.adaptive_solve(p, cfg)
for i in range(reps):
    torch.cuda.synchronize()
    print(f"=== e2e round {i}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    p.upload_async(A, b)
    rep = ihs.adaptive_solve(p, cfg)
    torch.cuda.synchronize()
    print(f"e2e round {i}: {1e3 * (time.perf_counter() - t0):.1f} ms, solve total_ms "
          f"{rep.device_times['total_ms']:.1f}", flush=True)
