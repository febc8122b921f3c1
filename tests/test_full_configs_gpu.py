"""Parity at the bench's own full-size configurations: C2 (Kinect 320x240
pair, 76,800 points) and C3 (HDL-32 LiDAR pair, 72,000 points), both
adaptive:3, against the reference's build_tree and register_clouds on the
same clouds (tests/golden/make_golden_full.py).  Bars as north_star."""
import os

import numpy as np
import pytest

from tests.helpers import GOLDEN, TREE_KEYS, rotation_angle_between

pytestmark = pytest.mark.gpu


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


def _load(name):
    tr = _tr()
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    g = {k: z[k] for k in z.files}
    gen = tr.kinect_pair if name.startswith("c2_") else tr.lidar_pair
    tg, sr, _ = gen(int(g["seed"]))
    assert np.array_equal(np.array([tg.sum(), np.abs(tg).sum(), float(len(tg))]), g["tg_sum"])
    assert np.array_equal(np.array([sr.sum(), np.abs(sr).sum(), float(len(sr))]), g["sr_sum"])
    g["tg"], g["sr"] = tg, sr
    g["tree"] = {k: g["tree_" + k] for k in TREE_KEYS}
    return g


def _relerr_rows(a, b):
    a = a.reshape(len(a), -1)
    b = b.reshape(len(b), -1)
    scale = np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    return float(np.max(np.linalg.norm(a - b, axis=1) / scale))


@pytest.mark.parametrize("name", ["c2_kinect77k_L3", "c3_lidar72k_L3"])
def test_full_size_tree(ctx, name):
    tr = _tr()
    g = _load(name)
    h = tr.build_tree(g["tg"], tr.ModelConfig(max_level=3), ctx=ctx).host()
    G = g["tree"]
    assert len(h["weight"]) == len(G["weight"])
    for k in ("parent", "first_child", "child_count", "level"):
        assert np.array_equal(h[k], G[k]), k
    assert _relerr_rows(h["weight"][:, None], G["weight"][:, None]) <= 1e-4
    assert np.abs(h["mean"] - G["mean"]).max() <= 1e-4 * np.abs(G["mean"]).max()
    # covariances and eigenvalues within 1e-4 relative, plus the rounding
    # floor of a scatter formed from raw moments (m2/m0 - mu mu^T): a leaf of
    # coincident points far from the origin (C3: |mu| ~ 50 m) has a
    # covariance that IS that noise clamped at the 1e-12 floor in both
    # implementations (as tests/test_random_sweep_gpu.py)
    cs = np.linalg.norm(G["cov"].reshape(len(G["cov"]), -1), axis=1)
    noise = 64 * np.finfo(float).eps * (np.sum(G["mean"] ** 2, axis=1) + cs)
    dc = np.linalg.norm((h["cov"] - G["cov"]).reshape(len(cs), -1), axis=1)
    assert np.all(dc <= 1e-4 * cs + noise), np.max(dc / np.maximum(cs, 1e-300))
    ls = np.linalg.norm(G["lambdas"], axis=1)
    dl = np.linalg.norm(h["lambdas"] - G["lambdas"], axis=1)
    assert np.all(dl <= 1e-4 * ls + noise)


@pytest.mark.parametrize("name", ["c2_kinect77k_L3", "c3_lidar72k_L3"])
def test_full_size_register(ctx, name):
    tr = _tr()
    g = _load(name)
    res = tr.register_clouds(g["tg"], g["sr"], tr.RegistrationConfig(variant=tr.Variant("adaptive", 3)), ctx)
    ext = float(np.linalg.norm(g["tg"].max(0) - g["tg"].min(0)))
    assert rotation_angle_between(res.transform.rotation, g["rc_R"]) <= 1e-4
    assert np.linalg.norm(res.transform.translation - g["rc_t"]) <= 1e-4 * ext
    assert res.converged == bool(g["rc_meta"][1])
    assert abs(res.iterations - int(g["rc_meta"][0])) <= 1
