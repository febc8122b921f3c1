"""C5 slice throughput vs pairs in flight (device-resident pairs)."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = tr.default_context()
pairs = [tr.kinect_pair(1 + k) for k in range(n)]
tg = [torch.from_numpy(p[0]).cuda() for p in pairs]
sr = [torch.from_numpy(p[1]).cuda() for p in pairs]
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
for s in [int(x) for x in sys.argv[2:]] or [4, 6, 8, 12]:
    tr.register_batch(tg, sr, cfg, ctx, s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = tr.register_batch(tg, sr, cfg, ctx, s)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"inflight {s:2d}: {n / dt:7.1f} reg/s  ({1e3 * dt / n:.2f} ms/pair, converged {sum(r.converged for r in res)})", flush=True)
