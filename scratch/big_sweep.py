"""Ad-hoc wide parity sweep (not part of the suite): random clouds vs the live reference."""
import sys, traceback, numpy as np
sys.path.insert(0, '.')
from tests.test_random_sweep_gpu import _cloud, test_random_cloud_parity
from oracle.oracle import Ref
from paper_1807_02587_b200 import treereg as tr
ref, ctx = Ref(), tr.default_context()
shapes = ("uniform", "blobs", "plane", "line", "duplicates", "mixed")
fails = 0
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for s in range(N):
    r = np.random.default_rng(50000 + s)
    n = int(r.integers(1, 20000)); sh = shapes[int(r.integers(0, 6))]; L = int(r.integers(1, 5))
    try:
        test_random_cloud_parity(ctx, ref, 5000 + s, n, sh, L)
    except Exception as e:
        fails += 1
        print("FAIL", s, n, sh, L, repr(e)[:300])
print("done", N, "fails", fails)
