"""Prints the device timeline of one C2 tree build (phase breakdown)."""
import sys, numpy as np, ctypes as C, collections
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
if len(sys.argv) > 1: ctx.set_sm_budget(int(sys.argv[1]))
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(2):
    d = None; tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), d, ctx)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.float64) / 1e3; lab = lab[:n]
o = np.argsort(t, kind="stable"); t = t[o]; lab = lab[o]
dt = np.diff(t)
groups = collections.OrderedDict()
for i in range(1, n):
    L = lab[i]
    if L >= 1000: key = f"calib stage {L % 10}"
    elif L >= 900: key = f"rematch {L}"
    else:
        r, ph = divmod(L, 100)
        key = f"round {r} {'reduce' if ph >= 50 else 'tiles '} phase {ph % 50}"
    groups.setdefault(key, []).append(dt[i-1])
tot = t[-1] - t[0]
print("total us", tot, d)
for k, v in groups.items():
    print(f"{k:32s} n={len(v):3d} sum={sum(v):9.1f} us  mean={np.mean(v):8.1f}")

agg = collections.OrderedDict()
for k, v in groups.items():
    kk = k.split(" phase")[0] if k.startswith("round") else k.split(" 9")[0]
    agg[kk] = agg.get(kk, 0) + sum(v)
for k, v in agg.items(): print(f"AGG {k:24s} {v:9.1f} us")
