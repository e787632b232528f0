"""One C4-Gaussian adaptive solve (n = 2^22, d = 2048, sigma_j = 1/j, nu = 1e-4, Gaussian, rho = 0.1) with the
streamed S: prints the m-schedule, iterations and per-phase device times."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2006_05874_b200 import ihs  # noqa: E402

n, d = 1 << 22, 2048
A = np.empty((n, d), order="F")
b = np.empty(n)
ihs.synth_generate(n, d, spectrum=1, decay=0.0, noise_std=0.01, data_seed=0, A_out=A, b_out=b)
p = ihs.ProblemInstance(A, b, 1e-4)
del A
cfg = ihs.SolverConfig(rho=0.1, sketch_kind=ihs.SketchKind.Gaussian, eps=1e-10, seed=0)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    t = time.perf_counter()
    r = ihs.adaptive_solve(p, cfg)
    dt = time.perf_counter() - t
    print(f"solve {rep}: {dt:.2f} s  converged={r.converged} iterations={r.iterations} rejections={r.rejections} "
          f"final_m={r.final_m} m={[e.m for e in r.log if int(e.branch) == 2]}", flush=True)
    print("  phases", {k: round(v, 1) for k, v in r.device_times.items() if k.endswith('_ms')}, flush=True)
