import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1807_02587_b200 import treereg as tr
ctx = tr.default_context()
for n in (50000, 200000, 1000000):
    tg = tr.synthetic("scene", n, 4)
    T = tr.random_rigid_transform(8.0, 0.03, 4)
    src = (tg - T.translation) @ T.rotation
    r = tr.register_clouds(tg, src, tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), ctx)
    err = np.degrees(np.arccos(np.clip((np.trace(r.transform.rotation.T @ T.rotation) - 1) / 2, -1, 1)))
    print(n, "iters", r.iterations, "conv", r.converged, "rot err", err, "crit", r.criterion_trace[:3], r.criterion_trace[-2:])
