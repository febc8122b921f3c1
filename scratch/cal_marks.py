import sys, os, numpy as np
sys.path.insert(0, '.')
os.environ["TRG_BUILD_DBG"] = "5"
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(3): tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.int64); lab = lab[:n]
t0 = t[lab == 1000 + 9 * 10 + 2][0]  # end of pass 9 = start of pass 10
print("n marks", n)
def rel(L): return (t[lab == L] - t0) / 1e3
for L in (1101, 5001, 5002, 5003, 5010, 5040, 5041, 5042, 5043, 5031, 5030, 5020, 1102):
    v = rel(L)
    if len(v): print(L, "count", len(v), "min %.2f med %.2f max %.2f us" % (v.min(), np.median(v), v.max()))
