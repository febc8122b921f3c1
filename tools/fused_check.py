"""Fused register_batch vs register_clouds: per pair, the first iteration
whose criterion / eval count differs (bit level)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
seeds = [int(x) for x in sys.argv[1:]] or [3, 4, 5, 6]
pairs = [tr.kinect_pair(k) for k in seeds]
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
ones = [tr.register_clouds(p[0], p[1], cfg, ctx) for p in pairs]
for inflight in (1, 2, 4):
    res = tr.register_batch([p[0] for p in pairs], [p[1] for p in pairs], cfg, ctx, inflight)
    for k, (r, o) in enumerate(zip(res, ones)):
        ev = [int(x) for x in r.eval_counts[:r.iterations]]
        eo = [int(x) for x in o.eval_counts[:o.iterations]]
        cb, co = np.asarray(r.criterion_trace[:r.iterations]), np.asarray(o.criterion_trace[:o.iterations])
        d_ev = next((i for i in range(min(len(ev), len(eo))) if ev[i] != eo[i]), None)
        d_cb = next((i for i in range(min(len(cb), len(co))) if cb[i] != co[i]), None)
        same = r.transform.rotation.tobytes() == o.transform.rotation.tobytes()
        print(f"inflight {inflight} pair {k}: it {r.iterations}/{o.iterations} same={same} "
              f"first ev diff {d_ev} first crit diff {d_cb} "
              f"crit0 {cb[0]!r} vs {co[0]!r}", flush=True)
