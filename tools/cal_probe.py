"""Fine marks of calibration pass 10 (library built with EXTRA=-DTRG_CAL_PROBE -DTRG_ASSOC_PROBE)."""
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


def show(t0, labels):
    for L in labels:
        v = np.sort(t[lab == L] - t0)
        if len(v):
            q = np.percentile(v, [0, 10, 50, 90, 100])
            print(L, "n", len(v), " ".join("%.2f" % x for x in q))


P = int(sys.argv[1]) if len(sys.argv) > 1 else 10
t1 = t[lab == 1000 + 10 * (P - 1) + 2][0] if P > 0 else t[lab == 902][0]
t0 = t[lab == 1000 + 10 * P + 1][0]
print("pass 10 stage-1 span %.2f us" % (t0 - t1))
show(t1, (5100, 5103, 5101, 5102))
print("pass 10 stage-2 span %.2f us" % (t[lab == 1000 + 10 * P + 2][0] - t0))
show(t0, (5000, 5001, 5002, 5003, 5010, 5011, 5030, 1102))
