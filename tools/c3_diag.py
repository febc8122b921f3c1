import sys
import numpy as np
sys.path.insert(0, ".")
from tests.test_full_configs_gpu import _load, _tr  # noqa: E402
tr = _tr()
g = _load(sys.argv[1] if len(sys.argv) > 1 else "c3_lidar72k_L3")
ctx = tr.Context(0)
h = tr.build_tree(g["tg"], tr.ModelConfig(max_level=3), ctx=ctx).host()
G = g["tree"]
a = h["cov"].reshape(len(h["cov"]), -1)
b = G["cov"].reshape(len(G["cov"]), -1)
err = np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-300)
o = np.argsort(-err)[:8]
for j in o:
    print(j, "lvl", G["level"][j], "cc", G["child_count"][j], "err %.3g" % err[j], "w %.4g/%.4g" % (h["weight"][j], G["weight"][j]),
          "lam", np.round(G["lambdas"][j], 6), "dmean %.3g" % np.abs(h["mean"][j] - G["mean"][j]).max())
print("nodes with err > 1e-4:", int((err > 1e-4).sum()), "of", len(err))
