"""Concurrency experiment: B contexts (streams) x B host threads, each
running register_clouds on its own C2 pair with an SM budget of 148/B."""
import sys, time, threading, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
import torch
pairs = [tr.kinect_pair(k) for k in range(1, 9)]
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
for B in (1, 2, 4, 8):
    for budget in ([148] if B == 1 else [148 // B]):
        ctxs = [tr.Context(0) for _ in range(B)]
        for c in ctxs: c.set_sm_budget(budget)
        devp = [(torch.from_numpy(p[0]).cuda(), torch.from_numpy(p[1]).cuda()) for p in pairs[:B]]
        def work(i, reps):
            for _ in range(reps):
                tr.register_clouds(devp[i][0], devp[i][1], cfg, ctxs[i])
        for reps, timed in ((1, False), (4, True)):
            th = [threading.Thread(target=work, args=(i, reps)) for i in range(B)]
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for t in th: t.start()
            for t in th: t.join()
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"B={B} budget={budget:3d}: {B*4/dt:7.1f} reg/s", flush=True)
        for c in ctxs: c.close()
