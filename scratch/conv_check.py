import sys, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
for k in list(range(1, 9)) + list(range(100, 108)):
    tg, sr, gt = tr.kinect_pair(k)
    r = tr.register_clouds(tg, sr, cfg)
    e = np.degrees(np.arccos(np.clip((np.trace(r.transform.rotation.T @ gt.rotation) - 1) / 2, -1, 1)))
    ang = np.degrees(np.arccos(np.clip((np.trace(gt.rotation) - 1) / 2, -1, 1)))
    print(k, "iters", r.iterations, "conv", r.converged, "rot err %.4f deg" % e, "gt rot %.2f deg |t| %.3f" % (ang, np.linalg.norm(gt.translation)), "crit", r.criterion_trace[-3:])
