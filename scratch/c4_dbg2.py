import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1807_02587_b200 import treereg as tr
from oracle.oracle import Port
ctx = tr.default_context()
n = 1000000
tg = tr.synthetic("scene", n, 4)
T = tr.random_rigid_transform(8.0, 0.03, 4)
src = (tg - T.translation) @ T.rotation
tree = tr.build_tree(tg, tr.ModelConfig(max_level=3), ctx=ctx)
diag = tr.bbox_diagonal(tg)
r = tr.register_with_tree(tree, src, tr.RegistrationConfig(max_em_iterations=5), diag)
print("gpu 5 iters crit", r.criterion_trace, r.transform.rotation_angle())
h = tree.host()
t0 = time.time()
o = Port().register_with_tree(h, src, max_iters=5, target_diag=diag)
print("port 5 iters crit", o["criterion_before"], time.time() - t0)
# association moments on the identity transform, GPU vs port
m = tr.associate_adaptive(src, tree, None, tr.AssocConfig(), with_m2=False)
mp = Port().associate(h, src, lambda_c=0.01)
print("assoc m0 max rel", np.max(np.abs(m.m0 - mp.m0) / np.maximum(mp.m0, 1e-300)), "sum", m.m0.sum(), mp.m0.sum(), m.outliers, mp.outliers)
