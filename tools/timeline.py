"""Device timeline of one C2 registration (globaltimer marks written by CTA 0
of the persistent kernels; labels in include/treereg_b200.h).  Prints the
time between consecutive marks grouped by stage.

    python tools/timeline.py [build|em]
"""
import collections
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1807_02587_b200 import _lib, treereg as tr  # noqa: E402


def marks(ctx):
    t = np.zeros(1024, np.uint64)
    lab = np.zeros(1024, np.int32)
    n = _lib.lib().trg_debug_build_timeline(ctx.h, t.ctypes.data_as(_lib.u64p),
                                            lab.ctypes.data_as(_lib.ip), 1024)
    t = t[:n].astype(np.float64) / 1e3
    lab = lab[:n]
    o = np.argsort(t, kind="stable")
    return t[o], lab[o]


def group(label):
    if 2000 <= label < 3000:
        return f"em stage {label % 10}"
    if 1000 <= label < 2000:
        return f"cal stage {label % 10}"
    if label < 900:
        r, ph = divmod(label, 100)
        return f"round {r} {'reduce' if ph >= 50 else 'tiles '} phase {ph % 50:2d}"
    return f"lab {label}"


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "build"
    ctx = tr.default_context()
    tg, sr, gt = tr.kinect_pair(2)
    tgd = torch.from_numpy(tg).cuda()
    srd = torch.from_numpy(sr).cuda()
    for _ in range(3):
        tree = tr.build_tree(tgd, tr.ModelConfig(max_level=3), None, ctx)
    if what == "em":
        diag = float(np.linalg.norm(tg.max(0) - tg.min(0)))
        for _ in range(3):
            res = tr.register_with_tree(tree, srd, tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), diag)
        print("iterations", res.iterations)
    t, lab = marks(ctx)
    print("marks", len(t), "span us %.1f" % (t[-1] - t[0]))
    g = collections.defaultdict(list)
    for i in range(1, len(t)):
        g[group(int(lab[i]))].append(t[i] - t[i - 1])
    for k, v in sorted(g.items()):
        print(f"{k:28s} n={len(v):3d} sum={sum(v):8.1f} mean={np.mean(v):7.2f} us")


if __name__ == "__main__":
    main()
