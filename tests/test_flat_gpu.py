"""Flat-mixture variant ("GMM J=n") on the GPU vs the
reference's own build_flat_gmm / responsibilities_dense / register_clouds
flat:J (golden fixtures from tests/golden/make_golden_flat.py).  Bars as
north_star: mixture parameters 1e-4 relative (the seeding is the
reference's own mt19937_64 stream, so the seeds are identical), dense
moments to rounding, transforms 1e-4 rad / 1e-4 x extent."""
import numpy as np
import pytest

from tests.helpers import flat_names, load_flat, rotation_angle_between

pytestmark = pytest.mark.gpu


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


def _relerr_rows(a, b):
    a = a.reshape(len(a), -1)
    b = b.reshape(len(b), -1)
    scale = np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    return np.linalg.norm(a - b, axis=1) / scale


@pytest.mark.parametrize("name", flat_names())
def test_flat_build_matches_reference(ctx, name):
    tr = _tr()
    g = load_flat(name)
    diag = tr.BuildDiagnostics()
    mix = tr.build_flat_gmm(g["points"], int(g["J"]), tr.ModelConfig(rng_seed=int(g["seed"])),
                            diag, ctx=ctx)
    h, G = mix.host(), g["mix"]
    # the flat fit's EM log-likelihood trace (gmm.cpp:729-734, BuildDiagnostics)
    assert len(diag.node_ll_traces) == 1
    ll = np.asarray(diag.node_ll_traces[0])
    assert ll.shape == g["ll_trace"].shape
    assert np.abs(ll - g["ll_trace"]).max() <= 1e-8 * np.abs(g["ll_trace"]).max()
    assert len(h["weight"]) == int(g["J"])
    assert np.array_equal(h["weight"] == 0.0, G["weight"] == 0.0)  # same dormant set
    live = G["weight"] > 0
    assert _relerr_rows(h["weight"][live, None], G["weight"][live, None]).max() <= 1e-4
    assert np.abs(h["mean"] - G["mean"]).max() <= 1e-4 * np.abs(G["mean"]).max()
    assert _relerr_rows(h["cov"], G["cov"]).max() <= 1e-4
    assert _relerr_rows(h["lambdas"], G["lambdas"]).max() <= 1e-4
    assert (h["level"] == 0).all() and (h["child_count"] == 0).all()


@pytest.mark.parametrize("name", flat_names())
def test_dense_moments_match_reference(ctx, name):
    tr = _tr()
    g = load_flat(name)
    mix = tr.GmmTree.from_host(g["mix"], ctx)
    for tag, T in (("id", tr.RigidTransform.identity()), ("pose", tr.RigidTransform(g["R"], g["t"]))):
        m = tr.responsibilities_dense(g["points"], mix, T)
        tp, outl, ev = g[f"dense_{tag}_counts"]
        assert (m.total_points, m.outliers, m.density_evaluations) == (tp, outl, ev)
        m0 = g[f"dense_{tag}_m0"]
        assert np.abs(m.m0 - m0).max() <= 1e-10 * max(1.0, m0.max())
        assert np.abs(m.m1 - g[f"dense_{tag}_m1"]).max() <= 1e-10 * max(1.0, np.abs(g[f"dense_{tag}_m1"]).max())
        assert np.abs(m.m2 - g[f"dense_{tag}_m2"]).max() <= 1e-10 * max(1.0, np.abs(g[f"dense_{tag}_m2"]).max())


@pytest.mark.parametrize("name", [n for n in flat_names() if not n.endswith("J512")])
def test_flat_register_matches_reference(ctx, name):
    tr = _tr()
    g = load_flat(name)
    cfg = tr.RegistrationConfig(variant=tr.Variant("flat", int(g["J"])))
    res = tr.register_clouds(g["points"], g["src"], cfg, ctx)
    ext = float(np.linalg.norm(g["points"].max(0) - g["points"].min(0)))
    assert rotation_angle_between(res.transform.rotation, g["rc_R"]) <= 1e-4
    assert np.linalg.norm(res.transform.translation - g["rc_t"]) <= 1e-4 * ext
    assert res.converged == bool(g["rc_meta"][1])
    assert res.model_components == int(g["J"])


def test_dense_on_tree_nodes(ctx):
    """responsibilities_dense also takes a tree's nodes as the component set
    (test_association.cpp:137, 167): every node, all levels."""
    tr = _tr()
    from tests.helpers import load_golden
    g = load_golden("scene3k_L3")
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    m = tr.responsibilities_dense(g["points"], tree)
    assert m.density_evaluations == len(g["points"]) * tree.size()
    assert abs(m.m0.sum() - (len(g["points"]) - m.outliers)) <= 1e-8 * len(g["points"])


def test_flat_errors(ctx):
    tr = _tr()
    g = load_flat("flat_blobs1k_J8")
    with pytest.raises(tr.InvalidArgument):
        tr.build_flat_gmm(g["points"], 0, ctx=ctx)
    with pytest.raises(tr.InvalidArgument):
        tr.build_flat_gmm(g["points"][:5], 6, ctx=ctx)
    bad = g["points"].copy()
    bad[3, 1] = np.inf
    with pytest.raises(tr.InvalidArgument):
        tr.build_flat_gmm(bad, 4, ctx=ctx)
    with pytest.raises(tr.InvalidArgument):
        tr.Variant.parse("flat:0")
