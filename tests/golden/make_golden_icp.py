"""Golden fixtures for the ICP point-to-point comparator:
the reference's register_clouds with variant icp (registration.cpp:211-298)
on three clouds, FROM THE REFERENCE ITSELF (oracle/_ref).

    make -C oracle ref && python tests/golden/make_golden_icp.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402


def main():
    ref = Ref()
    cases = [("icp_lumpy2k", ref.unit_normalized(ref.synthetic("lumpy", 2000, 1)), (5.0, 0.02, 1)),
             ("icp_scene3k", ref.synthetic("scene", 3000, 21), (4.0, 0.02, 3)),
             ("icp_blobs1k", ref.synthetic("blobs", 1000, 5), (3.0, 0.01, 5))]
    for name, pts, (rot, tr, seed) in cases:
        R, t = ref.random_rigid_transform(rot, tr, seed)
        src = pts @ R.T + t
        rc = ref.register_clouds(pts, src, variant="icp")
        np.savez_compressed(os.path.join(HERE, name + ".npz"), points=pts, src=src, rc_R=rc["R"],
                            rc_t=rc["t"], rc_meta=np.array([rc["iterations"], int(rc["converged"])]))
        print(name, rc["iterations"], rc["converged"])


if __name__ == "__main__":
    main()
