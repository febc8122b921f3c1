"""Point-sharded build / calibration / EM against the
reference's own results.  Local communicators run k shards of one cloud on
one GPU through exactly the segmented path a k-GPU NCCL run takes (segment
launches, all-reduce of the per-node records, all-gather of argmax seeds);
an NCCL communicator of world 1 covers the NCCL binding.  Bars as north_star:
tree structure identical, GMM parameters 1e-4 relative, transforms 1e-4 rad /
1e-4 x extent."""
import os

import numpy as np
import pytest

from tests.helpers import GOLDEN, TREE_KEYS, load_golden, rotation_angle_between

pytestmark = pytest.mark.gpu

CASES = ["scene3k_L3", "kinect4k_L3", "c1_lumpy10k_L2"]


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


def _split(pts, k):
    tr = _tr()
    out = []
    for r in range(k):
        lo, hi = tr.shard_bounds(len(pts), k, r)
        out.append(np.ascontiguousarray(pts[lo:hi]))
    return out


def _relerr_rows(a, b):
    a = a.reshape(len(a), -1)
    b = b.reshape(len(b), -1)
    scale = np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    return float(np.max(np.linalg.norm(a - b, axis=1) / scale))


def _check_tree(h, G):
    assert len(h["weight"]) == len(G["weight"])
    for k in ("parent", "first_child", "child_count", "level"):
        assert np.array_equal(h[k], G[k]), k
    assert _relerr_rows(h["weight"][:, None], G["weight"][:, None]) <= 1e-4
    assert np.abs(h["mean"] - G["mean"]).max() <= 1e-4 * np.abs(G["mean"]).max()
    assert _relerr_rows(h["cov"], G["cov"]) <= 1e-4
    assert _relerr_rows(h["lambdas"], G["lambdas"]) <= 1e-4


@pytest.mark.parametrize("shards", [1, 2, 3])
@pytest.mark.parametrize("name", CASES)
def test_sharded_build_matches_reference(ctx, name, shards):
    tr = _tr()
    g = load_golden(name)
    comm = tr.Comm.local(shards, ctx)
    d = tr.BuildDiagnostics()
    tree = tr.build_tree_sharded(_split(g["points"], shards), comm,
                                 tr.ModelConfig(max_level=int(g["max_level"])), d)
    _check_tree(tree.host(), g["tree"])
    assert d.entries_per_round[0] == len(g["points"])
    assert d.calibration_passes >= 1
    comm.close()


@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("name", CASES)
def test_sharded_register_matches_reference(ctx, name, shards):
    tr = _tr()
    g = load_golden(name)
    comm = tr.Comm.local(shards, ctx)
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", int(g["max_level"])))
    res = tr.register_clouds_sharded(_split(g["points"], shards), _split(g["src"], shards), comm, cfg)
    diag = float(g["reg_meta"][2])
    assert rotation_angle_between(res.transform.rotation, g["rc_R"]) <= 1e-4
    assert np.linalg.norm(res.transform.translation - g["rc_t"]) <= 1e-4 * diag
    assert res.converged == bool(g["rc_meta"][1])
    comm.close()


def test_sharded_matches_single_gpu_path(ctx):
    """Same cloud, 1 shard vs 4 shards vs the single-launch path."""
    tr = _tr()
    g = load_golden("kinect4k_L3")
    cfg = tr.ModelConfig(max_level=3)
    one = tr.build_tree(g["points"], cfg, ctx=ctx).host()
    comm = tr.Comm.local(4, ctx)
    four = tr.build_tree_sharded(_split(g["points"], 4), comm, cfg).host()
    _check_tree(four, one)
    comm.close()


def test_nccl_world_of_one(ctx):
    tr = _tr()
    g = load_golden("lumpy2k_L2")
    try:
        uid = tr.Comm.unique_id()
    except tr.CudaError as e:  # pragma: no cover - libnccl missing
        pytest.skip(str(e))
    comm = tr.Comm.nccl(0, 1, uid, ctx)
    assert (comm.rank, comm.world, comm.local_shards) == (0, 1, 1)
    tree = tr.build_tree_sharded([g["points"]], comm, tr.ModelConfig(max_level=2))
    _check_tree(tree.host(), g["tree"])
    res = tr.register_clouds_sharded([g["points"]], [g["src"]], comm,
                                     tr.RegistrationConfig(variant=tr.Variant("adaptive", 2)))
    assert rotation_angle_between(res.transform.rotation, g["rc_R"]) <= 1e-4
    comm.close()


def test_sharded_c4_full_size(ctx):
    """BASELINE C4 at full size (1M points, depth 4) on 2 shards."""
    tr = _tr()
    z = np.load(os.path.join(GOLDEN, "c4_scene1M_L4.npz"))
    G = {k: z["tree_" + k] for k in TREE_KEYS}
    pts = tr.synthetic("scene", 1_000_000, 4)
    comm = tr.Comm.local(2, ctx)
    tree = tr.build_tree_sharded(_split(pts, 2), comm, tr.ModelConfig(max_level=4))
    _check_tree(tree.host(), G)
    R, t = z["R"], z["t"]
    src = (pts - t) @ R
    res = tr.register_clouds_sharded(_split(pts, 2), _split(src, 2), comm,
                                     tr.RegistrationConfig(variant=tr.Variant("adaptive", 4)))
    ext = float(np.linalg.norm(pts.max(0) - pts.min(0)))
    assert res.iterations == int(z["rc_meta"][0])
    assert rotation_angle_between(res.transform.rotation, z["rc_R"]) <= 1e-4
    assert np.linalg.norm(res.transform.translation - z["rc_t"]) <= 1e-4 * ext
    comm.close()


def test_sharded_errors(ctx):
    tr = _tr()
    g = load_golden("scene3k_L3")
    comm = tr.Comm.local(2, ctx)
    with pytest.raises(tr.InvalidArgument):
        tr.build_tree_sharded([g["points"]], comm)  # 1 cloud for 2 shards
    bad = _split(g["points"], 2)
    bad[1] = bad[1].copy()
    bad[1][3, 0] = np.nan
    with pytest.raises(tr.InvalidArgument):
        tr.build_tree_sharded(bad, comm, tr.ModelConfig(max_level=3))
    with pytest.raises(tr.InvalidArgument):
        tr.Comm.local(0, ctx)
    comm.close()
