"""One C2 tree build after warm-up (the command ncu captures)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
srd = torch.from_numpy(sr).cuda()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(n):
    res = tr.register_clouds(tgd, srd, tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), ctx)
torch.cuda.synchronize()
print("iterations", res.iterations)
