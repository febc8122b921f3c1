"""Generates tests/golden/c4_scene1M_L4.npz FROM THE REFERENCE ITSELF
(oracle/_ref/libtreereg_ref.so), for BASELINE config C4:
synthetic_scene(1,000,000, seed 4), depth-4 tree, pose
random_rigid_transform({8 deg, 0.03, seed 4}, 0).

The 24 MB cloud is NOT stored: the GPU test regenerates it with
trg_synthetic (bit-exact restatement of the reference generator, checked by
tests/test_synth.py) and the fixture stores a checksum of it.  Stored: the
reference tree (4,680-node bound), its diagnostics, the associate_adaptive
moments at the identity pose (lambda_c = 0.01) and the register_clouds
result for adaptive:4.

    make -C oracle ref && python tests/golden/make_golden_c4.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import TREE_KEYS, Ref  # noqa: E402


def main():
    ref = Ref()
    pts = ref.synthetic("scene", 1_000_000, 4)
    R, t = ref.random_rigid_transform(8.0, 0.03, 4)
    src = (pts - t) @ R          # target = R src + t
    t0 = time.time()
    tree = ref.build_tree(pts, max_level=4)
    tb = time.time() - t0
    out = {"points_sum": np.array([pts.sum(), np.abs(pts).sum(), float(len(pts))]),
           "R": R, "t": t, "max_level": 4, "calibration_drift": tree["calibration_drift"]}
    for k in TREE_KEYS:
        out["tree_" + k] = tree[k]
    m = ref.associate(tree, pts, np.eye(3), np.zeros(3), 0.01)
    out["assoc_m0"], out["assoc_m1"], out["assoc_m2"] = m.m0, m.m1, m.m2
    out["assoc_counts"] = np.array([m.total_points, m.outliers, m.density_evaluations])
    t0 = time.time()
    rc = ref.register_clouds(pts, src, level=4)
    tr_ = time.time() - t0
    out["rc_R"], out["rc_t"] = rc["R"], rc["t"]
    out["rc_meta"] = np.array([rc["iterations"], int(rc["converged"]), tb, tr_])
    np.savez_compressed(os.path.join(HERE, "c4_scene1M_L4.npz"), **out)
    ang = np.degrees(np.arccos(np.clip((np.trace(rc["R"].T @ R) - 1) / 2, -1, 1)))
    print("c4 nodes", len(tree["weight"]), "build s", tb, "register s", tr_, "iters", rc["iterations"],
          "converged", rc["converged"], "rot err deg", ang)


if __name__ == "__main__":
    main()
