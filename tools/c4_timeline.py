"""Device timeline of one C4 build (1M points, L=4): per-round tile / reduce
time and the calibration stages (`phases`: per phase)."""
import collections
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from timeline import marks, group  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tg = tr.synthetic("scene", 1000000, 4)
tgd = torch.from_numpy(tg).cuda()
for _ in range(2):
    tree = tr.build_tree(tgd, tr.ModelConfig(max_level=4), None, ctx)
t, lab = marks(ctx)
per_phase = len(sys.argv) > 1 and sys.argv[1] == "phases"
g = collections.defaultdict(float)
for i in range(1, len(t)):
    k = group(int(lab[i]))
    if not per_phase:
        k = k.rsplit(" phase", 1)[0]
    g[k] += t[i] - t[i - 1]
print("span us %.0f" % (t[-1] - t[0]))
for k, v in sorted(g.items()):
    print(f"{k:24s} {v:10.0f} us")
