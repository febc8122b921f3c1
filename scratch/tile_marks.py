import sys, os, numpy as np
sys.path.insert(0, '.')
os.environ["TRG_BUILD_DBG"] = "6"
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(3): tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.int64); lab = lab[:n]
start = t[lab == 6000]
t0 = start.min()
fin = [(int(l) - 6100, (int(x) - t0) / 1e3) for l, x in zip(lab, t) if 6100 <= l < 6200]
ent = [int(l) - 200000 for l in lab if l >= 200000]
print("CTAs", len(fin), "start spread us", (start.max() - start.min()) / 1e3)
fin = np.array(fin)
for k in sorted(set(fin[:, 0])):
    v = fin[fin[:, 0] == k][:, 1]
    print("tiles", int(k), "CTAs", len(v), "finish min %.1f med %.1f max %.1f us" % (v.min(), np.median(v), v.max()))
print("entries per CTA: min", min(ent), "max", max(ent), "mean", np.mean(ent))
nxt = t[(lab == 204) | (lab == 254)]
print("barrier mark after tiles:", (t[lab == 204][0] - t0) / 1e3 if (lab == 204).any() else None)
