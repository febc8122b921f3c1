import sys, numpy as np
sys.path.insert(0, '.')
from tests.helpers import load_golden
from paper_1807_02587_b200 import treereg as tr
ctx = tr.default_context()
g = load_golden("kinect4k_L3")
tree = tr.GmmTree.from_host(g["tree"], ctx)
ms = tr.MomentSet(g["lc001_m0"], g["lc001_m1"], None, int(g["lc001_counts"][0]))
for _ in range(5): tr.solve_mstep(tr.make_virtual_points(ms, tree))
