"""Per-iteration anatomy of one C2 EM (k_register timeline marks)."""
import sys, numpy as np, collections
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda(); srd = torch.from_numpy(sr).cuda()
tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
diag = float(np.linalg.norm(tg.max(0) - tg.min(0)))
for _ in range(3):
    res = tr.register_with_tree(tree, srd, tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), diag)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.float64) / 1e3; lab = lab[:n]
o = np.argsort(t, kind="stable"); t = t[o]; lab = lab[o]
print("iterations", res.iterations, "marks", n, "span us", t[-1] - t[0])
g = collections.defaultdict(list)
for i in range(1, n):
    L = lab[i]
    if 2000 <= L < 3000: g[f"stage {L % 10}"].append(t[i] - t[i - 1])
    else: g[f"lab {L}"].append(t[i] - t[i - 1])
for k, v in sorted(g.items()): print(f"{k:12s} n={len(v):3d} sum={sum(v):8.1f} mean={np.mean(v):6.1f}")
