import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
import torch
pairs = [tr.kinect_pair(100 + k) for k in range(24)]
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
tg = [torch.from_numpy(p[0]).cuda() for p in pairs]
sr = [torch.from_numpy(p[1]).cuda() for p in pairs]
ctx = tr.Context(0)
for s in (1, 2, 3, 4, 5, 6, 8):
    tr.register_batch(tg, sr, cfg, ctx, s)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(2): res = tr.register_batch(tg, sr, cfg, ctx, s)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"streams {s}: {48/dt:.1f} reg/s  converged {sum(r.converged for r in res)}/24", flush=True)
