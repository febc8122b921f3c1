import sys, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
from tests.helpers import load_golden
g = load_golden("kinect4k_L3")
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
ctx = tr.Context(0)
rs = [tr.register_clouds(g["points"], g["src"], cfg, ctx) for _ in range(4)]
for r in rs: print("rc iters", r.iterations, r.converged, r.transform.translation)
tree = tr.build_tree(g["points"], tr.ModelConfig(max_level=3), ctx=ctx)
diag = tr.bbox_diagonal(g["points"])
for _ in range(2):
    r = tr.register_with_tree(tree, g["src"], cfg, diag); print("rwt dev-tree iters", r.iterations, r.converged, r.transform.translation)
t2 = tr.GmmTree.from_host(tree.host(), ctx)
r = tr.register_with_tree(t2, g["src"], cfg, diag); print("rwt uploaded iters", r.iterations, r.converged, r.transform.translation)
h1, h2 = tree.host(), t2.host()
for k in h1:
    if isinstance(h1[k], np.ndarray) and not np.array_equal(h1[k], h2[k]): print("tree field differs after round trip:", k)
