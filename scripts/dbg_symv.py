import numpy as np, sys
sys.path.insert(0, '.')
from paper_2006_05874_b200 import ihs
rng = np.random.default_rng(0)
for (m, d) in [(20, 16), (40, 12), (100, 64), (600, 512), (70, 40), (9, 8), (33, 33)]:
    SA = rng.standard_normal((m, d))
    s = ihs.SketchedSystem.factorize(SA, 0.7)
    g = rng.standard_normal(d)
    z = s.solve(g)
    ref = np.linalg.solve(SA.T @ SA + 0.49 * np.eye(d), g)
    print(m, d, s.kind(), np.linalg.norm(z - ref) / np.linalg.norm(ref))
