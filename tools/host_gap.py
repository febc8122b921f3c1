"""How much of a C2 registration's device-timed step is host issue time:
the same step with a ~2 ms GPU sleep queued first (the host's API calls
then overlap the sleep) versus without."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tg, sr, _ = tr.kinect_pair(2)
dev = torch.device("cuda", 0)
tgd, srd = torch.from_numpy(tg).to(dev), torch.from_numpy(sr).to(dev)
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
for _ in range(3):
    tr.register_clouds(tgd, srd, cfg, ctx)
torch.cuda.synchronize()
for mode in ("plain", "sleep-first"):
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode == "sleep-first":
            torch.cuda._sleep(4_000_000)  # the host issues the registration meanwhile
        a.record()
        tr.register_clouds(tgd, srd, cfg, ctx)
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{mode:12s} median {np.median(ts):.3f} ms")
