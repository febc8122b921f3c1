"""Times the standalone E-step kernels on the C2 target (device-resident)."""
import sys, time, numpy as np, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_1807_02587_b200 import treereg as tr, _lib
ctx = tr.default_context()
tg, sr, gt = tr.kinect_pair(2)
tgd = torch.from_numpy(tg).cuda()
tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), ctx=ctx)
stream = torch.cuda.ExternalStream(ctx.stream)
for lc, m2 in [(0.0, True), (0.01, False), (0.0, False)]:
    cfg = tr.AssocConfig(lambda_c=lc)
    for _ in range(3): tr.associate_adaptive(tgd, tree, None, cfg, with_m2=m2)
    ts = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); m = tr.associate_adaptive(tgd, tree, None, cfg, with_m2=m2); e1.record(stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"lambda_c {lc} m2 {m2}: {np.median(ts)*1e3:.1f} us (incl. D2H of moments), evals {m.density_evaluations}")
