import sys, numpy as np, ctypes as C
sys.path.insert(0, '.')
from tests.helpers import load_golden
from paper_1807_02587_b200 import treereg as tr, _lib
ctx = tr.default_context()
g = load_golden("blobs1k_L2"); t = g["tree"]
m0, m1, N = g["lc001_m0"], g["lc001_m1"], g["lc001_counts"][0]
ata = np.zeros((6,6)); atb=np.zeros(6); nv = 0
for j in range(len(m0)):
    if m0[j] <= 1e-8*N: continue
    nv += 1; pi = m0[j]/N; mu = m1[j]/m0[j]
    lam = t["lambdas"][j]; lf = 1e-6*lam[0]
    for l in range(3):
        lm = max(lam[l], lf); w = np.sqrt(pi/lm); n = t["axes"][j][:,l]
        row = np.concatenate([w*np.cross(mu,n), w*n]); ata += np.outer(row,row); atb += row * w * n.dot(t["mean"][j]-mu)
v = np.concatenate([ata[np.triu_indices(6)], atb])
out = np.zeros(16)
L = _lib.lib(); f = L.trg_debug_solve; f.argtypes = [C.c_void_p, _lib.dp, C.c_int, _lib.dp]
f(ctx.h, v.ctypes.data_as(_lib.dp), nv, out.ctypes.data_as(_lib.dp))
print("gpu", out[:8]); print("numpy", np.linalg.solve(ata, atb), np.linalg.cond(ata)); print("golden", g["solve_omega"], g["solve_translation"])
for rep in range(3):
    f(ctx.h, v.ctypes.data_as(_lib.dp), nv, out.ctypes.data_as(_lib.dp))
print("sweeps", out[8], "cycles", out[9], "us", out[9]/1950)
