import sys, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
from tests.helpers import GOLDEN, TREE_KEYS
z = np.load(GOLDEN + "/c4_scene1M_L4.npz"); G = {k: z["tree_" + k] for k in TREE_KEYS}
pts = tr.synthetic("scene", 1_000_000, 4)
d = tr.BuildDiagnostics()
h = tr.build_tree(pts, tr.ModelConfig(max_level=4), d).host()
print("J", len(h["weight"]), len(G["weight"]), "cal passes", d.calibration_passes, "drift", d.calibration_drift, "golden drift", float(z["calibration_drift"]))
for k in ("weight", "mean", "cov", "lambdas"):
    a = h[k].reshape(len(h[k]), -1); b = G[k].reshape(len(G[k]), -1)
    e = np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    o = np.argsort(-e)[:5]
    print(k, "worst", [(int(i), float("%.3g" % e[i]), int(G["level"][i]), int(G["child_count"][i]), float("%.3g" % G["weight"][i])) for i in o])
    print("   count >1e-4:", int((e > 1e-4).sum()), " >1e-6:", int((e > 1e-6).sum()), " >1e-9:", int((e > 1e-9).sum()))
