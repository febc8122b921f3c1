import sys, time, threading, numpy as np
sys.path.insert(0, '.')
from paper_1807_02587_b200 import treereg as tr
import torch
pairs = [tr.kinect_pair(k) for k in range(1, 5)]
cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
devp = [(torch.from_numpy(p[0]).cuda(), torch.from_numpy(p[1]).cuda()) for p in pairs]
for budget in (148, 74, 37, 18):
    c = tr.Context(0); c.set_sm_budget(budget)
    for _ in range(2): tr.register_clouds(devp[0][0], devp[0][1], cfg, c)
    t0 = time.perf_counter()
    for _ in range(5): r = tr.register_clouds(devp[0][0], devp[0][1], cfg, c)
    print(f"B=1 budget {budget}: {(time.perf_counter()-t0)/5*1e3:.2f} ms/reg, build {r.model_build_seconds*1e3:.2f} em {r.em_seconds*1e3:.2f}", flush=True)
    c.close()
ctxs = [tr.Context(0) for _ in range(2)]
for c in ctxs: c.set_sm_budget(74)
T0 = time.perf_counter()
log = []
def work(i):
    for _ in range(3):
        a = time.perf_counter(); tr.register_clouds(devp[i][0], devp[i][1], cfg, ctxs[i]); b = time.perf_counter()
        log.append((i, (a-T0)*1e3, (b-T0)*1e3))
for _ in range(2):
    T0 = time.perf_counter(); log.clear()
    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th: t.start()
    for t in th: t.join()
for e in sorted(log, key=lambda x: x[1]): print("thread %d  %.2f -> %.2f ms" % e)
from paper_1807_02587_b200 import _lib
for i, c in enumerate(ctxs):
    t = np.zeros(1024, np.uint64); lab = np.zeros(1024, np.int32)
    n = _lib.lib().trg_debug_build_timeline(c.h, t.ctypes.data_as(_lib.u64p), lab.ctypes.data_as(_lib.ip), 1024)
    t = t[:n]; lab = lab[:n]
    o = np.argsort(t); t = t[o]; lab = lab[o]
    base = int(t[0]) if i == 0 else base
    print(i, "marks", n, "first", (int(t[0]) - base) / 1e3, "last", (int(t[-1]) - base) / 1e3, "us")
    sel = [k for k in range(n) if lab[k] in (100, 150, 200, 250, 900, 1001, 1391, 1392)]
    print("   ", [(int(lab[k]), round((int(t[k]) - base) / 1e3, 1)) for k in sel][:12])
