"""EM time, FP64 parity mode vs FP32 fast scoring (C2 and C4 register_with_tree)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
for name in ("c2", "c4"):
    if name == "c2":
        tg, sr, _ = tr.kinect_pair(2)
        L = 3
    else:
        tg = tr.synthetic("scene", 1000000, 4)
        T = tr.random_rigid_transform(8.0, 0.03, 4)
        sr = T(tg)
        L = 4
    tgd, srd = torch.from_numpy(tg).cuda(), torch.from_numpy(sr).cuda()
    tree = tr.build_tree(tgd, tr.ModelConfig(max_level=L), None, ctx)
    diag = float(np.linalg.norm(tg.max(0) - tg.min(0)))
    for fast in (False, True):
        cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", L), fast_scoring=fast)
        tr.register_with_tree(tree, srd, cfg, diag)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            r = tr.register_with_tree(tree, srd, cfg, diag)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        print(f"{name} fast={fast}: {1e3 * dt:.3f} ms per EM ({r.iterations} iterations, "
              f"{1e3 * dt / r.iterations:.3f} ms/iter), em_seconds {1e3 * r.em_seconds:.3f} ms")
