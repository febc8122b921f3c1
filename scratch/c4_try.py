import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1807_02587_b200 import treereg as tr
ctx = tr.default_context()
tg = tr.synthetic("scene", 1000000, 4)
T = tr.random_rigid_transform(8.0, 0.03, 4)
src = T.inverse()(tg)
tgd = torch.from_numpy(tg).cuda(); srd = torch.from_numpy(src).cuda()
for L in (3, 4):
    d = tr.BuildDiagnostics()
    t0 = time.time(); tree = tr.build_tree(tgd, tr.ModelConfig(max_level=L), d, ctx); torch.cuda.synchronize(); t1 = time.time()
    print("L", L, "build s", round(t1 - t0, 3), "nodes", tree.size(), "E", d.entries_per_round, "K", d.expanded_per_round, "cal", d.calibration_passes)
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", L))
    t0 = time.time(); r = tr.register_clouds(tgd, srd, cfg, ctx); t1 = time.time()
    err = np.degrees(np.arccos(np.clip((np.trace(r.transform.rotation.T @ T.rotation) - 1) / 2, -1, 1)))
    print("  register_clouds s", round(t1 - t0, 3), "build", r.model_build_seconds, "em", r.em_seconds, "iters", r.iterations, "conv", r.converged, "rot err deg", err)
