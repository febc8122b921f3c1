"""Reduce-phase marks of the barrier schedule (EXTRA=-DTRG_RP_PROBE=<phase>, TRG_DF=0):
node 0's item reductions (7000+10r), its node update start/end (7001/7002)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import torch  # noqa: E402
from timeline import marks  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(3):
    tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t, lab = marks(ctx)
P = int(sys.argv[1])
for r in range(3):
    t0 = t[lab == r * 100 + P][0]      # end of the tile pass (after grid_sync)
    t1 = t[lab == r * 100 + 50 + P][0]  # end of the reduce phase
    red = np.sort(t[lab == 7000 + 10 * r] - t0)
    print("round", r, "reduce phase %.2f us" % (t1 - t0),
          "item done pct 0/50/100: %s" % (np.percentile(red, [0, 50, 100]).round(2) if len(red) else "-"),
          "update %.2f -> %.2f" % tuple((t[lab == 7001 + 10 * r][0] - t0, t[lab == 7002 + 10 * r][0] - t0)))
# inside the update of node 0 (round r): 7100 start, 7110/7111 around the SIMT
# eigensolve, 7101/7102 around the M-steps
for r in range(3):
    a, b = t[lab == 7001 + 10 * r][0], t[lab == 7002 + 10 * r][0]
    m = (t >= a) & (t <= b) & (lab >= 7100)
    print("round", r, " ".join("%d:%.2f" % (l, x - a) for l, x in zip(lab[m], t[m])))
# raw SM cycles of the M-step eigensolve (label 7199 carries cycles, not ns)
t2 = np.zeros(1024, np.uint64)
l2 = np.zeros(1024, np.int32)
from paper_1807_02587_b200 import _lib  # noqa: E402
n = _lib.lib().trg_debug_build_timeline(ctx.h, t2.ctypes.data_as(_lib.u64p), l2.ctypes.data_as(_lib.ip), 1024)
print("eig cycles", t2[:n][l2[:n] == 7199][:12])
