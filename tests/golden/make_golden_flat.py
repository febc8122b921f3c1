"""Golden fixtures for the flat-mixture variant ("GMM J=n")
FROM THE REFERENCE ITSELF (oracle/_ref/libtreereg_ref.so): build_flat_gmm
(gmm.cpp:659-736), responsibilities_dense (association.cpp:54-89) and
register_clouds with variant flat:J (registration.cpp:191-202).

    make -C oracle ref && python tests/golden/make_golden_flat.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import TREE_KEYS, Ref  # noqa: E402


def cases(ref):
    lumpy = ref.unit_normalized(ref.synthetic("lumpy", 2000, 1))
    yield "flat_lumpy2k_J16", lumpy, 16, 0, (15.0, 0.05, 1)
    yield "flat_scene3k_J64", ref.synthetic("scene", 3000, 21), 64, 7, (8.0, 0.03, 3)
    yield "flat_blobs1k_J8", ref.synthetic("blobs", 1000, 5), 8, 3, (8.0, 0.03, 5)
    # the acceptance criterion's dense model size (acceptance_main.cpp:305)
    yield "flat_lumpy5k_J512", ref.unit_normalized(ref.synthetic("lumpy", 5000, 2)), 512, 0, (15.0, 0.05, 2)


def main():
    ref = Ref()
    for name, pts, J, seed, (rot, tr, pseed) in cases(ref):
        mix = ref.build_flat_gmm(pts, J, seed=seed)
        R, t = ref.random_rigid_transform(rot, tr, pseed)
        out = {"points": pts, "J": J, "seed": seed, "R": R, "t": t, "ll_trace": mix["ll_trace"]}
        for k in TREE_KEYS:
            out["mix_" + k] = mix[k]
        for tag, (RR, tt) in (("id", (np.eye(3), np.zeros(3))), ("pose", (R, t))):
            m = ref.responsibilities_dense(mix, pts, RR, tt)
            out[f"dense_{tag}_m0"], out[f"dense_{tag}_m1"], out[f"dense_{tag}_m2"] = m.m0, m.m1, m.m2
            out[f"dense_{tag}_counts"] = np.array([m.total_points, m.outliers, m.density_evaluations])
        src = pts @ R.T + t
        out["src"] = src
        if J <= 64:
            rc = ref.register_clouds(pts, src, level=J, variant="flat")
            out["rc_R"], out["rc_t"] = rc["R"], rc["t"]
            out["rc_meta"] = np.array([rc["iterations"], int(rc["converged"])])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, len(pts), "J", J, "ll", mix["ll_trace"][-1], flush=True)


if __name__ == "__main__":
    main()
