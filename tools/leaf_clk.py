import sys
import numpy as np
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr, _lib  # noqa: E402
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t = np.zeros(1024, np.uint64)
lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
first = t[512:].astype(np.int64)
second = lab[512:].astype(np.int64)
m = (first > 0) & (first < 10**9)
print("n", m.sum())
print("cycles A pct 10/50/90/max", np.percentile(first[m], [10, 50, 90, 100]))
print("cycles B pct 10/50/90/max", np.percentile(second[m], [10, 50, 90, 100]))
