"""One wave of `n` C2-style pairs through the fused register_batch (after a
warm-up wave), for launch lists / ncu captures of k_build / k_calibrate /
k_em_tree in batch mode."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ctx = tr.default_context()
pairs = [tr.kinect_pair(1 + k) for k in range(n)]
tg = [torch.from_numpy(p[0]).cuda() for p in pairs]
sr = [torch.from_numpy(p[1]).cuda() for p in pairs]
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
tr.register_batch(tg, sr, cfg, ctx, n)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = tr.register_batch(tg, sr, cfg, ctx, n)
torch.cuda.synchronize()
print(f"wave of {n}: {1e3 * (time.perf_counter() - t0):.2f} ms, iterations {[r.iterations for r in res]}")
print("build s", [round(r.model_build_seconds * 1e3, 2) for r in res][:4], "em s", [round(r.em_seconds * 1e3, 2) for r in res][:4])
