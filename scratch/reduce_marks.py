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
def at(L): return (t[lab == L][0]) if (lab == L).any() else None
t0 = at(4)  # round 0 phase 4 reduce end mark (54) ... use tile mark of phase 5
base = at(5)
for L in (5, 7001, 7002, 55, 6):
    v = at(L)
    print(L, None if v is None else "%.2f us" % ((v - base) / 1e3))
