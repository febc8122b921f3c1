"""Shared test helpers (numpy only; no oracle imports)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TREE_KEYS = ("weight", "mean", "cov", "lambdas", "axes", "log_norm", "parent", "first_child",
             "child_count", "level")


def golden_names():
    """Tree fixtures that carry their input cloud (c2_/c3_/c4_* regenerate
    theirs; flat_* are the flat-mixture fixtures)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("c2_", "c3_", "c4_", "flat_", "seq_", "icp_")))


def flat_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "flat_*.npz")))


def load_flat(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    g = {k: z[k] for k in z.files}
    g["mix"] = {k: g["mix_" + k] for k in TREE_KEYS}
    g["mix"]["max_level"] = 1
    return g


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    g = {k: z[k] for k in z.files}
    g["tree"] = {k: g["tree_" + k] for k in TREE_KEYS}
    g["tree"]["max_level"] = int(g["max_level"])
    return g


def log_scores(tree, y, nodes):
    """log(w * N(y; node)) per node, as log w + log_norm - q/2 (gmm.cpp:37-47)."""
    out = []
    for j in nodes:
        w = tree["weight"][j]
        if not w > 0:
            out.append(-np.inf)
            continue
        d = y - tree["mean"][j]
        p = tree["axes"][j].T @ d
        q = np.sum(p * p / tree["lambdas"][j])
        out.append(np.log(w) + tree["log_norm"][j] - 0.5 * q)
    return np.array(out)


def near_tie_on_path(tree, y, lambda_c, tol=1e-6):
    """True if, along the best-path walk of y, some level's top-two sibling
    log-scores are within `tol` (the documented near-tie rule), or a
    complexity test sits within `tol` of lambda_c."""
    top = int(np.sum(tree["level"] == 0))
    first, count, node = 0, top, -1
    for _ in range(int(tree["max_level"])):
        ls = log_scores(tree, y, range(first, first + count))
        if len(ls) >= 2:
            s = np.sort(ls)[::-1]
            if np.isfinite(s[0]) and s[0] - s[1] <= tol * max(1.0, abs(s[0])):
                return True
        node = first + int(np.argmax(ls))
        if tree["child_count"][node] == 0:
            break
        lam = tree["lambdas"][node]
        c = lam[2] / lam.sum()
        if abs(c - lambda_c) <= tol:
            return True
        if c <= lambda_c:
            break
        first, count = int(tree["first_child"][node]), int(tree["child_count"][node])
    return False


def rel_err(a, b, floor=1e-300):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))) if a.size else 0.0


def rotation_angle_between(Ra, Rb):
    c = np.clip((np.trace(Ra.T @ Rb) - 1.0) * 0.5, -1.0, 1.0)
    return float(np.arccos(c))
