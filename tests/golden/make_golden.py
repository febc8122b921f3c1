"""Generates the golden fixtures in tests/golden/*.npz FROM THE REFERENCE
ITSELF (oracle/_ref/libtreereg_ref.so = /root/reference/proj/core/src built
with the test shims).  Run here (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture holds the input cloud, the reference's build_tree output, its
associate_adaptive moments and per-point deposits at three lambda_c values,
one make_virtual_points+solve_mstep solution, and a register_with_tree
result.  The GPU tests compare against these files, so they need neither
/root/reference nor the oracle build at run time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import TREE_KEYS, Ref  # noqa: E402


def cases(ref):
    lumpy = ref.unit_normalized(ref.synthetic("lumpy", 2000, 1))
    yield "lumpy2k_L2", lumpy, 2, (15.0, 0.05, 1)
    yield "scene3k_L3", ref.synthetic("scene", 3000, 21), 3, (8.0, 0.03, 3)
    yield "blobs1k_L2", ref.synthetic("blobs", 1000, 5), 2, (8.0, 0.03, 5)
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1807_02587_b200 import treereg  # host-side generator only
    tg, _, _ = treereg.kinect_pair(2)
    yield "kinect4k_L3", np.ascontiguousarray(tg[::19][:4000]), 3, (5.0, 0.05, 2)
    # BASELINE config C1: unit_normalized(synthetic_lumpy(10000, 1)), L = 2,
    # pose random_rigid_transform({15 deg, 0.05, seed 1}, 0)
    yield "c1_lumpy10k_L2", ref.unit_normalized(ref.synthetic("lumpy", 10000, 1)), 2, (15.0, 0.05, 1)


def main():
    ref = Ref()
    for name, pts, L, (rot, tr, seed) in cases(ref):
        tree = ref.build_tree(pts, max_level=L)
        R, t = ref.random_rigid_transform(rot, tr, seed)
        out = {"points": pts, "R": R, "t": t, "max_level": L,
               "calibration_drift": tree["calibration_drift"]}
        for k in TREE_KEYS:
            out["tree_" + k] = tree[k]
        out["ll_trace_root"] = tree["ll_traces"][0]
        for tag, lc in (("lc0", 0.0), ("lc001", 0.01), ("lc13", 1.0 / 3.0)):
            m = ref.associate(tree, pts, R, t, lc)
            node, w = ref.associate_points(tree, pts, R, t, lc)
            out[f"{tag}_m0"], out[f"{tag}_m1"], out[f"{tag}_m2"] = m.m0, m.m1, m.m2
            out[f"{tag}_counts"] = np.array([m.total_points, m.outliers, m.density_evaluations])
            out[f"{tag}_node"], out[f"{tag}_w"] = node, w
        m = ref.associate(tree, pts, R, t, 0.01)
        s = ref.solve_mstep(tree, m.m0, m.m1, m.total_points)
        for k in ("omega", "translation", "R", "t"):
            out["solve_" + k] = s[k]
        out["solve_scalars"] = np.array([s["criterion_before"], s["criterion_after"],
                                         s["condition"], s["n_vps"]])
        src = pts @ R.T + t
        diag = ref.bbox_diagonal(pts)
        reg = ref.register_with_tree(tree, src, target_diag=diag)
        out["src"] = src
        out["reg_R"], out["reg_t"] = reg["R"], reg["t"]
        out["reg_meta"] = np.array([reg["iterations"], int(reg["converged"]), diag])
        out["reg_crit_before"], out["reg_crit_after"] = reg["criterion_before"], reg["criterion_after"]
        out["reg_evals"] = reg["eval_counts"]
        rc = ref.register_clouds(pts, src, level=L)
        out["rc_R"], out["rc_t"] = rc["R"], rc["t"]
        out["rc_meta"] = np.array([rc["iterations"], int(rc["converged"])])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, len(pts), "nodes", len(tree["weight"]), "reg iters", reg["iterations"],
              "converged", reg["converged"])


if __name__ == "__main__":
    main()
