import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_random_sweep_gpu import _cloud, CASES
from oracle.oracle import Ref
from paper_1807_02587_b200 import treereg as tr
ref = Ref(); ctx = tr.default_context()
for seed, n, shape, L in CASES:
    if shape != "mixed": continue
    pts = _cloud(shape, n, np.random.default_rng(seed))
    G = ref.build_tree(pts, max_level=L)
    h = tr.build_tree(pts, tr.ModelConfig(max_level=L), ctx=ctx).host()
    cs = np.linalg.norm(G["cov"].reshape(len(G["cov"]), -1), axis=1)
    dn = np.linalg.norm((h["cov"] - G["cov"]).reshape(len(cs), -1), axis=1)
    r = dn / np.maximum(cs, 1e-300)
    j = int(np.argmax(r))
    print(seed, n, L, "J", len(cs), "worst node", j, "rel", r[j], "level", G["level"][j], "children", G["child_count"][j],
          "w", G["weight"][j], "cov", G["cov"][j].ravel()[:3], "gpu", h["cov"][j].ravel()[:3], "lam", G["lambdas"][j], h["lambdas"][j],
          "mean", G["mean"][j], "drift", G["calibration_drift"])
    bad = np.nonzero(r > 1e-6)[0]
    print("  nodes > 1e-6:", bad[:20], r[bad[:20]])
