"""Print the raw mark sequence (label, +us since previous) between two labels."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import torch  # noqa: E402
from timeline import marks  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

a, b = int(sys.argv[1]), int(sys.argv[2])
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
for _ in range(3):
    tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
t, lab = marks(ctx)
i0 = int(np.nonzero(lab == a)[0][0])
i1 = int(np.nonzero(lab == b)[0][0])
for i in range(i0, i1 + 1):
    print(int(lab[i]), "%+.2f" % (t[i] - t[i - 1]))
