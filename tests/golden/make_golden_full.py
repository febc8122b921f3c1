"""Full-size golden fixtures for the bench configurations C2 (320x240 Kinect
frame pair, 76,800 points, adaptive:3) and C3 (HDL-32 LiDAR sweep pair,
72,000 points, adaptive:3), FROM THE REFERENCE ITSELF
(oracle/_ref/libtreereg_ref.so).  The clouds are not stored: the GPU test
regenerates them with the product's frame-pair generators
(trg_synth_kinect_pair / trg_synth_lidar_pair, deterministic host code) and
checks a checksum.

    make -C oracle ref && python tests/golden/make_golden_full.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import TREE_KEYS, Ref  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402  (host generators only)


def main():
    ref = Ref()
    for name, gen, seed in (("c2_kinect77k_L3", tr.kinect_pair, 2), ("c3_lidar72k_L3", tr.lidar_pair, 3)):
        tg, sr, gt = gen(seed)
        t0 = time.time()
        tree = ref.build_tree(tg, max_level=3)
        rc = ref.register_clouds(tg, sr, level=3)
        out = {"seed": seed, "max_level": 3,
               "tg_sum": np.array([tg.sum(), np.abs(tg).sum(), float(len(tg))]),
               "sr_sum": np.array([sr.sum(), np.abs(sr).sum(), float(len(sr))]),
               "calibration_drift": tree["calibration_drift"],
               "rc_R": rc["R"], "rc_t": rc["t"], "rc_meta": np.array([rc["iterations"], int(rc["converged"])])}
        for k in TREE_KEYS:
            out["tree_" + k] = tree[k]
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, len(tg), "nodes", len(tree["weight"]), "iters", rc["iterations"], rc["converged"],
              "%.1fs" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main()
