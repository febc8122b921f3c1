import sys, numpy as np, ctypes as C
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(2): tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), ctx=ctx)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.float64)/1e3; lab = lab[:n]
t0 = t[lab == 4999][0]
starts = {l-5000: v for l, v in zip(lab, t) if 5000 <= l < 6000}
ends = {l-6000: v for l, v in zip(lab, t) if 6000 <= l < 7000}
nxt = t[(t > t0) & (lab < 1000)]
print("phase reduce start ->", "end barrier mark at", (nxt.min() - t0) if len(nxt) else None)
d = [(starts[k]-t0, ends[k]-starts[k]) for k in sorted(starts)]
st = np.array([x[0] for x in d]); du = np.array([x[1] for x in d])
print("node update start (us after phase start): min %.1f med %.1f max %.1f" % (st.min(), np.median(st), st.max()))
print("node update duration (us): min %.1f med %.1f max %.1f" % (du.min(), np.median(du), du.max()))
ms = {l-8000: v for l, v in zip(lab, t) if 8000 <= l < 8100}
me = {l-8100: v for l, v in zip(lab, t) if 8100 <= l < 8200}
du2 = np.array([me[k]-ms[k] for k in ms if k in me])
pre = np.array([ms[k]-starts[k] for k in ms if k in starts])
print("M-step part (us): min %.1f med %.1f max %.1f; before M-step: med %.1f" % (du2.min(), np.median(du2), du2.max(), np.median(pre)))
