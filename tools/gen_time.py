"""Host generator vs device renderer for the C2 pair (wall clock, after warm-up)."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.default_context()
tr.kinect_pair_device(1, ctx)
torch.cuda.synchronize()
for name, fn in (("host kinect_pair", lambda k: tr.kinect_pair(k)),
                 ("device kinect_pair_device", lambda k: tr.kinect_pair_device(k, ctx)),
                 ("host lidar_pair", lambda k: tr.lidar_pair(k)),
                 ("device lidar_pair_device", lambda k: tr.lidar_pair_device(k, ctx))):
    t0 = time.perf_counter()
    for k in range(20):
        fn(k)
    torch.cuda.synchronize()
    print(f"{name:28s} {1e3 * (time.perf_counter() - t0) / 20:7.2f} ms per pair")
