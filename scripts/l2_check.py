# bit-exactness of the SRHT sketch at 9..12 high bits (n_pad 2^19..2^22) against the oracle; run with
# IHS_SRHT_L2=0/1 and IHS_SRHT_L2_NS=k to cover each path
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2006_05874_b200 import ihs
from oracle import oracle as O
rng = np.random.default_rng(3)
for n, d, ms in [((1 << 19) - 5, 5, (3, 400, 60000)), ((1 << 20) + 0, 4, (1000,)), ((1 << 21) - 3, 3, (7, 70000)),
                 ((1 << 22) - 3, 3, (9, 131072)), ((1 << 22), 2, (100000,))]:
    A = np.asfortranarray(rng.standard_normal((n, d)))
    for m in ms:
        ok = np.array_equal(ihs.srht_sketch(A, m, 5 + m), O.srht_sketch(A, m, 5 + m))
        print(n, d, m, ok, flush=True)
        assert ok
print('ok')
