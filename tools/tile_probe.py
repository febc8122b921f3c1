"""SM-clock marks inside CTA 0's tiles of one build phase (library built with
EXTRA=-DTRG_TILE_PROBE=<phase> [-DTRG_TILE_PROBE_ROUND=<round>]), cycles from
the tile start: context + bulk copies landed (2), warp 0's log-density loop
start / end (5 / 6), log-densities done (3), responsibilities done (4), warp
0's moment loop done (7), tile done (9).  Clocks in shared memory, no
atomics inside the tile."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import _lib, treereg as tr  # noqa: E402

ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(3):
    tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t = np.zeros(1024, np.uint64)
lab = np.zeros(1024, np.int32)
n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
t, lab = t[:n], lab[:n]
m = (lab >= 8100) & (lab < 8200)
print(" ".join("%d:%d" % (l - 8100, x) for l, x in zip(lab[m], t[m]) if l != 8108))
