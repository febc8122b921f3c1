"""Anatomy of one round-2 reduce phase (TRG_BUILD_DBG=7)."""
import sys, os, numpy as np
sys.path.insert(0, '.')
os.environ["TRG_BUILD_DBG"] = "7"
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(3): tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.int64); lab = lab[:n]
t0 = t[lab == 6999].min()
print("n marks", n)
for L in (6999, 7100, 7200, 7000, 255):
    v = (t[lab == L] - t0) / 1e3
    if len(v): print(L, "count", len(v), "min %.2f p10 %.2f med %.2f p90 %.2f max %.2f us" % (v.min(), np.percentile(v, 10), np.median(v), np.percentile(v, 90), v.max()))
