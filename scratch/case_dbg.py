import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_random_sweep_gpu import _cloud
from tests.helpers import near_tie_on_path, rel_err, rotation_angle_between
from oracle.oracle import Ref
from paper_1807_02587_b200 import treereg as tr
ref, ctx = Ref(), tr.default_context()
seed, n, shape, L = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
pts = _cloud(shape, n, np.random.default_rng(seed))
G = ref.build_tree(pts, max_level=L)
h = tr.build_tree(pts, tr.ModelConfig(max_level=L), ctx=ctx).host()
print("J", len(h["weight"]), len(G["weight"]))
for k in ("parent", "first_child", "child_count", "level"):
    print(k, np.array_equal(h[k], G[k]))
print("weight", np.abs(h["weight"] - G["weight"]).max())
print("mean", np.abs(h["mean"] - G["mean"]).max(), np.abs(G["mean"]).max())
cs = np.linalg.norm(G["cov"].reshape(len(G["cov"]), -1), axis=1)
dc = np.linalg.norm((h["cov"] - G["cov"]).reshape(len(cs), -1), axis=1)
print("cov rel", (dc / cs).max(), "w", G["weight"], "\n gpu w", h["weight"])
R, t = ref.random_rigid_transform(5.0, 0.05, seed)
tree = tr.GmmTree.from_host(G, ctx)
_, node, w = tr.associate_adaptive(pts, tree, tr.RigidTransform(R, t), tr.AssocConfig(lambda_c=0.01), per_point=True)
rnode, rw = ref.associate_points(G, pts, R, t, lambda_c=0.01)
bad = np.nonzero(node != rnode)[0]
print("assoc mismatches", len(bad))
ok = node == rnode
print("w relerr", rel_err(w[ok], rw[ok]))
src = (pts - t) @ R
var = "tree" if seed % 2 else "adaptive"
want = ref.register_clouds(pts, src, level=L, variant=var)
got = tr.register_clouds(pts, src, tr.RegistrationConfig(variant=tr.Variant(var, L)), ctx)
print("reg", rotation_angle_between(got.transform.rotation, want["R"]), np.abs(got.transform.rotation - want["R"]).max(),
      np.linalg.norm(got.transform.translation - want["t"]), got.iterations, want["iterations"], got.converged, want["converged"])
