"""Hash of the C2 tree and registration (bit-identity check across refactors)."""
import hashlib
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
for cfg in ("c2", "c3"):
    tg, sr, _ = tr.kinect_pair(2) if cfg == "c2" else tr.lidar_pair(3)
    t = tr.build_tree(tg, tr.ModelConfig(max_level=3), ctx=ctx).host()
    h = hashlib.sha1()
    for k in ("weight", "mean", "cov", "lambdas", "axes", "log_norm", "parent", "level"):
        h.update(np.ascontiguousarray(t[k]).tobytes())
    r = tr.register_clouds(tg, sr, tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), ctx)
    h2 = hashlib.sha1(np.ascontiguousarray(r.transform.rotation).tobytes() +
                      np.ascontiguousarray(r.transform.translation).tobytes()).hexdigest()
    print(cfg, "tree", h.hexdigest()[:16], "J", len(t["weight"]), "reg", h2[:16], "it", r.iterations)
