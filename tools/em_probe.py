"""EM solver-CTA marks (library built with EXTRA=-DTRG_EM_PROBE): per
iteration, the time from the workers' arrival (stage 1 end) to the node loop
end (7100), the block reduction (7101), the 6x6 solve (7102) and the publish
(stage 3 end)."""
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
srd = torch.from_numpy(sr).cuda()
tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
diag = float(np.linalg.norm(tg.max(0) - tg.min(0)))
for _ in range(3):
    res = tr.register_with_tree(tree, srd, tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), diag)
t, lab = marks(ctx)
print("iterations", res.iterations)
for i in range(len(t)):
    if 7000 <= lab[i] < 7200 or 2000 <= lab[i] < 3000:
        print(int(lab[i]), "%.2f" % (t[i] - t[0]))
