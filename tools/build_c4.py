"""One C4 tree build after a warm-up (the command ncu captures)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tg = tr.synthetic("scene", 1000000, 4)
tgd = torch.from_numpy(tg).cuda()
for _ in range(2):
    tree = tr.build_tree(tgd, tr.ModelConfig(max_level=4), None, ctx)
torch.cuda.synchronize()
print("nodes", tree.size())
