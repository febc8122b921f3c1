"""Randomised parity sweep against the live reference (oracle/_ref, the
reference's own sources): ragged sizes around the 32-point expansion gate
and the 256-entry tile (1, 9, 31-33, 255-257, 1023, 3001, 4097), shapes
that stress the covariance floor (lines, planes, duplicate points, mixed
scales) and depths 1-3.  Per case: build_tree (structure exact, parameters
1e-4), per-point association on the reference's tree (node ids equal except
documented near-ties, path weights 1e-12) and register_clouds (1e-4 rad /
1e-4 x extent)."""
import numpy as np
import pytest

from tests.helpers import near_tie_on_path, rel_err, rotation_angle_between

pytestmark = pytest.mark.gpu


def _cloud(shape, n, rng):
    if shape == "uniform":
        return rng.uniform(-1, 1, size=(n, 3))
    if shape == "blobs":
        c = rng.normal(size=(4, 3)) * 2.0
        return c[rng.integers(0, 4, n)] + rng.normal(size=(n, 3)) * 0.2
    if shape == "plane":
        u = rng.uniform(-1, 1, size=(n, 2))
        return np.c_[u, 0.3 * u[:, 0] + 1e-3 * rng.normal(size=n)]
    if shape == "line":
        s = rng.uniform(-2, 2, size=n)
        return np.c_[s, 0.5 * s, -s] + 1e-4 * rng.normal(size=(n, 3))
    if shape == "duplicates":
        base = rng.normal(size=(max(1, n // 8), 3))
        return base[rng.integers(0, len(base), n)]
    if shape == "mixed":  # far-apart clusters at very different scales
        a = rng.normal(size=(n // 2, 3)) * 1e-2
        b = rng.normal(size=(n - n // 2, 3)) * 5.0 + 40.0
        return np.r_[a, b]
    raise ValueError(shape)


CASES = [(1, 1, "uniform", 2), (2, 9, "blobs", 2), (3, 31, "plane", 2), (4, 32, "uniform", 2),
         (5, 33, "line", 3), (6, 255, "duplicates", 2), (7, 256, "blobs", 3), (8, 257, "plane", 3),
         (9, 1023, "mixed", 3), (10, 3001, "uniform", 2), (11, 4097, "blobs", 1),
         (12, 2500, "line", 3)]
# plus drawn cases: size, shape and depth from the seed
_SHAPES = ("uniform", "blobs", "plane", "line", "duplicates", "mixed")
for _s in range(13, 37):
    _r = np.random.default_rng(1000 + _s)
    CASES.append((_s, int(_r.integers(1, 6000)), _SHAPES[int(_r.integers(0, 6))], int(_r.integers(1, 4))))


@pytest.mark.parametrize("seed,n,shape,L", CASES)
def test_random_cloud_parity(ctx, ref, seed, n, shape, L):
    from paper_1807_02587_b200 import treereg as tr
    rng = np.random.default_rng(seed)
    pts = _cloud(shape, n, rng)
    # build_tree
    G = ref.build_tree(pts, max_level=L)
    h = tr.build_tree(pts, tr.ModelConfig(max_level=L), ctx=ctx).host()
    assert len(h["weight"]) == len(G["weight"])
    for k in ("parent", "first_child", "child_count", "level"):
        assert np.array_equal(h[k], G[k]), k
    assert np.abs(h["weight"] - G["weight"]).max() <= 1e-4 * max(1.0, G["weight"].max())
    scale = max(np.abs(G["mean"]).max(), 1e-300)
    assert np.abs(h["mean"] - G["mean"]).max() <= 1e-4 * scale
    # covariances within 1e-4 relative, plus the rounding floor of a scatter
    # formed from raw moments (m2/m0 - mu mu^T): eps * |mu|^2 per entry.  A leaf
    # holding one point (or duplicates) far from the origin has a covariance
    # that IS that rounding noise clamped at the 1e-12 floor in both
    # implementations ("mixed" clouds at |x| ~ 50: 1e-13 of noise on 1e-12).
    cs = np.linalg.norm(G["cov"].reshape(len(G["cov"]), -1), axis=1)
    noise = 64 * np.finfo(float).eps * (np.sum(G["mean"] ** 2, axis=1) + cs)
    dc = np.linalg.norm((h["cov"] - G["cov"]).reshape(len(cs), -1), axis=1)
    assert np.all(dc <= 1e-4 * cs + noise), np.max(dc / np.maximum(cs, 1e-300))
    # per-point association on the reference's tree, under a small motion
    R, t = ref.random_rigid_transform(5.0, 0.05, seed)
    tree = tr.GmmTree.from_host(G, ctx)
    lc = 0.01
    _, node, w = tr.associate_adaptive(pts, tree, tr.RigidTransform(R, t), tr.AssocConfig(lambda_c=lc),
                                       per_point=True)
    rnode, rw = ref.associate_points(G, pts, R, t, lambda_c=lc)
    y = pts @ R.T + t
    for i in np.nonzero(node != rnode)[0]:
        assert near_tie_on_path(G, y[i], lc), f"point {i}: {node[i]} vs {rnode[i]}"
    ok = node == rnode
    # path weights: products of sibling posteriors; exp differs from the host
    # libm's by an ulp, which thin (line-like) components amplify to ~1e-12
    assert rel_err(w[ok], rw[ok]) <= 1e-10
    # register_clouds end to end (source = target moved by the inverse motion)
    if n >= 32:
        src = (pts - t) @ R
        var = "tree" if seed % 2 else "adaptive"  # tree:L = lambda_c 0 (full-depth walks)
        want = ref.register_clouds(pts, src, level=L, variant=var)
        got = tr.register_clouds(pts, src, tr.RegistrationConfig(variant=tr.Variant(var, L)), ctx)
        diag = float(np.linalg.norm(pts.max(0) - pts.min(0)))
        ang = rotation_angle_between(got.transform.rotation, want["R"])
        assert ang <= 1e-4 or np.abs(got.transform.rotation - want["R"]).max() <= 1e-6
        assert np.linalg.norm(got.transform.translation - want["t"]) <= 1e-4 * max(diag, 1e-12)


# ModelConfig away from the defaults (gmm.hpp:34-41): EM iterations per node,
# the expansion gate, both covariance regularisers, and depths up to 4.
CONFIGS = [dict(em_iters=1, min_points=32, eps=1e-4, abs_floor=1e-12, L=3),
           dict(em_iters=3, min_points=100, eps=1e-4, abs_floor=1e-12, L=3),
           dict(em_iters=12, min_points=8, eps=1e-4, abs_floor=1e-12, L=2),
           dict(em_iters=8, min_points=32, eps=1e-2, abs_floor=1e-12, L=3),
           dict(em_iters=8, min_points=32, eps=0.0, abs_floor=1e-6, L=3),
           dict(em_iters=5, min_points=16, eps=1e-3, abs_floor=1e-9, L=4)]


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_model_config_parity(ctx, ref, ci):
    from paper_1807_02587_b200 import treereg as tr
    c = CONFIGS[ci]
    pts = _cloud(("blobs", "plane", "uniform", "line", "mixed", "blobs")[ci], 4000,
                 np.random.default_rng(100 + ci))
    G = ref.build_tree(pts, max_level=c["L"], em_iters=c["em_iters"], min_points=c["min_points"],
                       eps=c["eps"], abs_floor=c["abs_floor"])
    mc = tr.ModelConfig(em_iterations_per_node=c["em_iters"], min_points_per_node=c["min_points"],
                        cov_regularization_epsilon=c["eps"], cov_regularization_absolute=c["abs_floor"],
                        max_level=c["L"])
    d = tr.BuildDiagnostics()
    h = tr.build_tree(pts, mc, d, ctx).host()
    assert len(h["weight"]) == len(G["weight"])
    for k in ("parent", "first_child", "child_count", "level"):
        assert np.array_equal(h[k], G[k]), k
    assert np.abs(h["weight"] - G["weight"]).max() <= 1e-4
    assert np.abs(h["mean"] - G["mean"]).max() <= 1e-4 * max(np.abs(G["mean"]).max(), 1e-300)
    cs = np.linalg.norm(G["cov"].reshape(len(G["cov"]), -1), axis=1)
    noise = 64 * np.finfo(float).eps * (np.sum(G["mean"] ** 2, axis=1) + cs)
    dc = np.linalg.norm((h["cov"] - G["cov"]).reshape(len(cs), -1), axis=1)
    assert np.all(dc <= 1e-4 * cs + noise)
    # BuildDiagnostics::node_ll_traces: one (em_iters + 1)-long trace per expansion
    assert len(d.node_ll_traces) == len(G["ll_traces"])
    for a, b in zip(d.node_ll_traces, G["ll_traces"]):
        assert len(a) == len(b) == c["em_iters"] + 1
        assert np.abs(np.asarray(a) - b).max() <= 1e-6 * max(1.0, np.abs(b).max())


# RegistrationConfig away from the defaults (registration.hpp:27-36): early
# stop by the iteration cap, tight / loose tolerances, lambda_c levels, the
# tree:L variant, the target-diagonal fallback (tree_extent_estimate).
REGS = [dict(variant="adaptive", lc=0.01, iters=3, rtol=1e-5, ttol=1e-5, diag=True),
        dict(variant="adaptive", lc=0.2, iters=50, rtol=1e-8, ttol=1e-8, diag=True),
        dict(variant="adaptive", lc=0.0, iters=50, rtol=1e-3, ttol=1e-3, diag=True),
        dict(variant="tree", lc=0.0, iters=20, rtol=1e-5, ttol=1e-5, diag=False),
        dict(variant="adaptive", lc=1.0 / 3.0, iters=50, rtol=1e-5, ttol=1e-5, diag=False)]


@pytest.mark.parametrize("ri", range(len(REGS)))
def test_registration_config_parity(ctx, ref, ri):
    from paper_1807_02587_b200 import treereg as tr
    c = REGS[ri]
    rng = np.random.default_rng(200 + ri)
    pts = _cloud(("blobs", "plane", "uniform", "blobs", "line")[ri], 3000, rng)
    G = ref.build_tree(pts, max_level=3)
    R, t = ref.random_rigid_transform(10.0, 0.1, 200 + ri)
    src = (pts - t) @ R
    diag = float(np.linalg.norm(pts.max(0) - pts.min(0))) if c["diag"] else 0.0
    want = ref.register_with_tree(G, src, variant=c["variant"], lambda_c=c["lc"], max_iters=c["iters"],
                                  rot_tol=c["rtol"], trans_tol=c["ttol"], target_diag=diag)
    cfg = tr.RegistrationConfig(variant=tr.Variant(c["variant"], 3), lambda_c=c["lc"],
                                max_em_iterations=c["iters"], rotation_tol=c["rtol"],
                                translation_tol=c["ttol"])
    got = tr.register_with_tree(tr.GmmTree.from_host(G, ctx), src, cfg, diag)
    assert got.iterations == want["iterations"]
    assert got.converged == want["converged"]
    assert np.abs(got.transform.rotation - want["R"]).max() <= 1e-6
    assert np.linalg.norm(got.transform.translation - want["t"]) <= 1e-6 * max(1.0, np.abs(pts).max())
    n = got.iterations
    assert np.array_equal(np.asarray(got.eval_counts[:n]), want["eval_counts"][:n])


@pytest.mark.parametrize("seed,n,shape,var,param", [(301, 3000, "blobs", "flat", 8), (302, 1500, "plane", "flat", 16),
                                                    (303, 800, "uniform", "icp", 0), (304, 2000, "mixed", "icp", 0)])
def test_flat_and_icp_random(ctx, ref, seed, n, shape, var, param):
    # (ICP on collinear points is ill-posed: the reference's own Kabsch
    # iterates to non-rotations there, so no parity is defined for it)
    from paper_1807_02587_b200 import treereg as tr
    pts = _cloud(shape, n, np.random.default_rng(seed))
    R, t = ref.random_rigid_transform(6.0, 0.05, seed)
    src = (pts - t) @ R
    want = ref.register_clouds(pts, src, level=param, variant=var)
    got = tr.register_clouds(pts, src, tr.RegistrationConfig(variant=tr.Variant(var, param)), ctx)
    assert got.iterations == want["iterations"]
    assert got.converged == want["converged"]
    assert np.abs(got.transform.rotation - want["R"]).max() <= 1e-6
    assert np.linalg.norm(got.transform.translation - want["t"]) <= 1e-6 * max(1.0, np.abs(pts).max())


def test_register_clouds_run_to_run_identical(ctx):
    """The whole queued register_clouds (bbox -> build -> EM, side-stream
    source copy) is bit-reproducible run to run, like the reference."""
    from paper_1807_02587_b200 import treereg as tr
    tg, sr, _ = tr.kinect_pair(3)
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    a = tr.register_clouds(tg, sr, cfg, ctx)
    b = tr.register_clouds(tg, sr, cfg, ctx)
    assert np.array_equal(a.transform.rotation, b.transform.rotation)
    assert np.array_equal(a.transform.translation, b.transform.translation)
    assert a.iterations == b.iterations
    assert np.array_equal(np.asarray(a.eval_counts[:a.iterations]), np.asarray(b.eval_counts[:b.iterations]))
