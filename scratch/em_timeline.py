import sys, numpy as np, ctypes as C, collections
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda(); srd = torch.from_numpy(sr).cuda()
tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), ctx=ctx)
for _ in range(2): res = tr.register_with_tree(tree, srd, tr.RegistrationConfig(), tr.bbox_diagonal(tg))
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.float64)/1e3; lab = lab[:n]
o = np.argsort(t); t = t[o]; lab = lab[o]
g = collections.defaultdict(list)
for i in range(1, n):
    g[lab[i] % 10].append(t[i] - t[i-1])
names = {0: "P3 tail (crit/state) + loop", 1: "P1 assoc + barrier", 2: "P2 combine + barrier", 3: "P3 fold + solve"}
print("iterations", res.iterations, "total us", t[-1] - t[0])
for k in sorted(g): print(names.get(k, k), "mean %.1f us" % np.mean(g[k]), "n", len(g[k]))
d = collections.defaultdict(list)
for i in range(1, n):
    if lab[i] in (7000, 7001, 7002, 7003): d[lab[i]].append(t[i] - t[i-1])
for k in sorted(d): print(k, "mean %.1f us" % np.mean(d[k]))
