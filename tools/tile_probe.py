"""Marks inside CTA 0's tiles of one build phase (library built with
EXTRA=-DTRG_TILE_PROBE=<phase> [-DTRG_TILE_PROBE_ROUND=<round>]): phase start
(8000), per tile: start (8001), context + bulk copies landed (8002),
log-densities done (8003), responsibilities done (8004), tile done (8009)."""
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
m = (lab >= 8000) & (lab < 8100)
t0 = t[m][0]
print(" ".join("%d:%.2f" % (l, x - t0) for l, x in zip(lab[m], t[m])))
