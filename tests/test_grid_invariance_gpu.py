"""Grid invariance (the reference's thread-count invariance, parallel.hpp:30-33):
the tree, the calibration and the registration must not depend on how many
SMs / CTAs the persistent kernels run on.  Every reduction on the path is
either in a fixed order that depends only on the data (tile records summed in
tile order) or exact (fixed-point association deposits, trg_fx.cuh), so the
results are compared BITWISE across SM budgets 148 / 74 / 37, and between
register_batch (SM-budgeted concurrent workers) and register_clouds."""
import numpy as np
import pytest

from tests.helpers import load_golden

pytestmark = pytest.mark.gpu

FIELDS = ("weight", "mean", "cov", "lambdas", "axes", "log_norm", "parent", "first_child",
          "child_count", "level")


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


def _tree_bytes(tree):
    h = tree.host()
    return {k: np.ascontiguousarray(h[k]).tobytes() for k in FIELDS}


def _reg_key(r):
    return (np.ascontiguousarray(r.transform.rotation).tobytes(),
            np.ascontiguousarray(r.transform.translation).tobytes(), r.iterations, r.converged)


@pytest.mark.parametrize("name,L", [("kinect4k_L3", 3), ("scene3k_L3", 3), ("lumpy2k_L2", 2),
                                    ("c2", 3)])
def test_bitwise_across_sm_budgets(name, L):
    tr = _tr()
    if name == "c2":  # BASELINE C2, full size (76,800 points per frame)
        tg, sr, _ = tr.kinect_pair(2)
        g = {"points": tg, "src": sr}
    else:
        g = load_golden(name)
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", L))
    trees, regs = [], []
    for budget in (0, 74, 37):
        ctx = tr.Context(0)
        if budget:
            ctx.set_sm_budget(budget)
        trees.append(_tree_bytes(tr.build_tree(g["points"], tr.ModelConfig(max_level=L), ctx=ctx)))
        regs.append(_reg_key(tr.register_clouds(g["points"], g["src"], cfg, ctx)))
        ctx.close()
    for t in trees[1:]:
        for k in FIELDS:
            assert t[k] == trees[0][k], f"tree field {k} depends on the SM budget"
    for r in regs[1:]:
        assert r == regs[0], "registration depends on the SM budget"


def test_bitwise_batch_vs_single(ctx):
    tr = _tr()
    pairs = [tr.kinect_pair(k) for k in (3, 4, 5, 6)]
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    res = tr.register_batch([p[0] for p in pairs], [p[1] for p in pairs], cfg, ctx, 4)
    for (t, s, _), r in zip(pairs, res):
        one = tr.register_clouds(t, s, cfg, ctx)
        assert _reg_key(r) == _reg_key(one)


@pytest.mark.parametrize("inflight", [2, 5, 16])
def test_bitwise_fused_batch_waves(ctx, inflight):
    """register_batch's fused path (tree variants): waves of `inflight` pairs,
    each wave's builds and EMs as single launches with one CTA group per pair
    (2: three waves 2 + 2 + 1; 5: one wave; 16: one wave of 5 on big groups)
    -- every pair bit-identical to its own register_clouds, eval counts
    included."""
    tr = _tr()
    pairs = [tr.kinect_pair(k) for k in (3, 4, 5, 6, 7)]
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    res = tr.register_batch([p[0] for p in pairs], [p[1] for p in pairs], cfg, ctx, inflight)
    for (t, s, _), r in zip(pairs, res):
        one = tr.register_clouds(t, s, cfg, ctx)
        assert _reg_key(r) == _reg_key(one)
        assert list(r.eval_counts) == list(one.eval_counts)
        assert np.array_equal(r.criterion_trace, one.criterion_trace)


def test_fused_batch_entry_overflow_retry():
    """A fresh context sizes the entry buffers for L <= 3 growth (12 x N); a
    depth-4 build outgrows them: the pair that overflowed is re-run alone
    with the grown buffers, and the batch still equals register_clouds."""
    tr = _tr()
    names = ["scene3k_L3", "kinect4k_L3", "lumpy2k_L2"]
    gs = [load_golden(n) for n in names]
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 4))
    ctx = tr.Context(0)
    try:
        res = tr.register_batch([g["points"] for g in gs], [g["src"] for g in gs], cfg, ctx, 3)
    finally:
        ctx.close()
    ctx1 = tr.Context(0)
    try:
        for g, r in zip(gs, res):
            assert _reg_key(r) == _reg_key(tr.register_clouds(g["points"], g["src"], cfg, ctx1))
    finally:
        ctx1.close()


@pytest.mark.parametrize("variant", [("adaptive", 3), ("tree", 2)])
def test_fused_batch_mixed_sizes_host_inputs(ctx, variant):
    """One wave of clouds of different sizes (3k / 4k / 10k / 76.8k points),
    host (numpy) inputs, both tree variants: every pair bit-identical to its
    own register_clouds."""
    tr = _tr()
    gs = [load_golden(n) for n in ("scene3k_L3", "kinect4k_L3", "blobs1k_L2")]
    tgs = [g["points"] for g in gs]
    srs = [g["src"] for g in gs]
    lt = tr.unit_normalized(tr.synthetic("lumpy", 10000, 1))
    tgs.append(lt)
    srs.append(tr.random_rigid_transform(15.0, 0.05, 1)(lt))
    kt, ks, _ = tr.kinect_pair(9)
    tgs.append(kt)
    srs.append(ks)
    cfg = tr.RegistrationConfig(variant=tr.Variant(*variant))
    res = tr.register_batch(tgs, srs, cfg, ctx, 5)
    for t, s, r in zip(tgs, srs, res):
        one = tr.register_clouds(t, s, cfg, ctx)
        assert _reg_key(r) == _reg_key(one)
        assert list(r.eval_counts) == list(one.eval_counts)
