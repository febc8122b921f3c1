"""Hash of the C4 tree (1M points, L=4) and its registration (bit-identity check)."""
import hashlib
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tg = tr.synthetic("scene", 1000000, 4)
T = tr.random_rigid_transform(8.0, 0.03, 4)
sr = T(tg)
t = tr.build_tree(tg, tr.ModelConfig(max_level=4), ctx=ctx).host()
h = hashlib.sha1()
for k in ("weight", "mean", "cov", "lambdas", "axes", "log_norm", "parent", "level"):
    h.update(np.ascontiguousarray(t[k]).tobytes())
r = tr.register_clouds(tg, sr, tr.RegistrationConfig(variant=tr.Variant("adaptive", 4)), ctx)
h2 = hashlib.sha1(np.ascontiguousarray(r.transform.rotation).tobytes() +
                  np.ascontiguousarray(r.transform.translation).tobytes()).hexdigest()
print("c4 tree", h.hexdigest()[:16], "J", len(t["weight"]), "reg", h2[:16], "it", r.iterations,
      "build %.1f ms em %.1f ms" % (1e3 * r.model_build_seconds, 1e3 * r.em_seconds))
