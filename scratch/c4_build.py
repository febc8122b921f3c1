"""One C4 tree build (synthetic_scene 1M, L=4): timeline per round/stage, for ncu too."""
import sys, collections, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr, _lib
import torch
ctx = tr.default_context()
pts = tr.synthetic("scene", 1_000_000, 4)
d = torch.from_numpy(pts).cuda()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(reps):
    diag = tr.BuildDiagnostics()
    tree = tr.build_tree(d, tr.ModelConfig(max_level=4), diag, ctx)
t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t = t[:n].astype(np.float64) / 1e3; lab = lab[:n]
o = np.argsort(t, kind="stable"); t = t[o]; lab = lab[o]
agg = collections.OrderedDict()
for i in range(1, n):
    L = lab[i]
    if L >= 1000: k = f"calib stage {L % 10}"
    elif L >= 900: k = "rematch"
    else:
        r, ph = divmod(L, 100)
        k = f"round {r} {'reduce' if ph >= 50 else 'tiles'}"
    agg[k] = agg.get(k, 0) + t[i] - t[i - 1]
print("total us", t[-1] - t[0], "E", list(diag.entries_per_round))
for k, v in agg.items(): print(f"{k:20s} {v:10.1f}")
