import sys, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
from tests.helpers import rotation_angle_between as ang
frames, gt = tr.kinect_sequence(11, 5, 2.0, 0.02)
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
for k in range(1, 5):
    link = gt[k - 1].inverse() * gt[k]
    r = tr.register_clouds(frames[k - 1], frames[k], cfg)
    print(k, "gt link rot %.2f deg" % np.degrees(ang(link.rotation, np.eye(3))), "err %.3f deg" % np.degrees(ang(r.transform.rotation, link.rotation)),
          "err vs inverse %.3f" % np.degrees(ang(r.transform.rotation, link.rotation.T)), r.iterations, r.converged)
