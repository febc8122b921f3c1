"""trg_register_batch (BASELINE config C5: independent frame pairs; tree
variants as waves of single launches with one CTA group per pair) against the reference's own
register_clouds results (golden fixtures) and against one-pair calls.
Tolerances as north_star: 1e-4 rad rotation, 1e-4 x extent translation."""
import numpy as np
import pytest

from tests.helpers import load_golden, rotation_angle_between

pytestmark = pytest.mark.gpu

L3 = ["scene3k_L3", "kinect4k_L3"]


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


@pytest.mark.parametrize("streams", [1, 2, 3])
def test_batch_matches_reference(ctx, streams):
    tr = _tr()
    gs = [load_golden(n) for n in L3] * 2  # 4 pairs, each fixture twice
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    res = tr.register_batch([g["points"] for g in gs], [g["src"] for g in gs], cfg, ctx, streams)
    assert len(res) == len(gs)
    for g, r in zip(gs, res):
        diag = float(g["reg_meta"][2])
        assert rotation_angle_between(r.transform.rotation, g["rc_R"]) <= 1e-4
        assert np.linalg.norm(r.transform.translation - g["rc_t"]) <= 1e-4 * diag
        assert r.converged == bool(g["rc_meta"][1])
    # the same pair twice in one batch: same answer to rounding
    for a, b in zip(res[:2], res[2:]):
        assert np.abs(a.transform.rotation - b.transform.rotation).max() <= 1e-12


def test_batch_device_resident_kinect_pairs(ctx):
    torch = pytest.importorskip("torch")
    tr = _tr()
    pairs = [tr.kinect_pair(k) for k in (3, 4, 5)]
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    tg = [torch.from_numpy(p[0]).cuda() for p in pairs]
    sr = [torch.from_numpy(p[1]).cuda() for p in pairs]
    res = tr.register_batch(tg, sr, cfg, ctx, 3)
    for (t, s, gt), r in zip(pairs, res):
        one = tr.register_clouds(t, s, cfg, ctx)
        assert rotation_angle_between(r.transform.rotation, one.transform.rotation) <= 1e-6
        assert np.abs(r.transform.translation - one.transform.translation).max() <= 1e-7
        assert r.converged == one.converged and r.iterations == one.iterations


def test_batch_errors(ctx):
    tr = _tr()
    g = load_golden("scene3k_L3")
    bad = g["src"].copy()
    bad[7, 1] = np.nan
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    with pytest.raises(tr.InvalidArgument, match="pair 1"):
        tr.register_batch([g["points"]] * 3, [g["src"], bad, g["src"]], cfg, ctx, 2)
    with pytest.raises(tr.InvalidArgument):
        tr.register_batch([g["points"]], [g["src"]], cfg, ctx, 25)  # > 24 pairs in flight
    with pytest.raises(tr.InvalidArgument):  # flat / ICP: <= 16 worker threads
        tr.register_batch([g["points"]], [g["src"]], tr.RegistrationConfig(variant=tr.Variant("icp", 0)),
                          ctx, 17)
    assert tr.register_batch([], [], cfg, ctx) == []


def test_register_sequence_matches_reference(ctx):
    """Frame-to-frame sequence: every link and the chained
    trajectory against the reference's register_clouds on the same frames
    (tests/golden/make_golden_seq.py); each link also equals a one-pair call."""
    import os
    from tests.helpers import GOLDEN
    tr = _tr()
    z = np.load(os.path.join(GOLDEN, "seq_kinect5.npz"))
    frames, gt = tr.kinect_sequence(11, 5, step_rot_deg=2.0, step_trans=0.02)
    assert np.array_equal(np.array([[f.sum(), np.abs(f).sum()] for f in frames]), z["frames_sum"])
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    res, traj = tr.register_sequence(frames, cfg, ctx, streams=2)
    assert len(res) == 4 and len(traj) == 5
    ext = float(np.linalg.norm(frames[0].max(0) - frames[0].min(0)))
    for k, r in enumerate(res):
        assert rotation_angle_between(r.transform.rotation, z["link_R"][k]) <= 1e-4
        assert np.linalg.norm(r.transform.translation - z["link_t"][k]) <= 1e-4 * ext
        assert r.converged == bool(z["link_meta"][k][1])
        one = tr.register_clouds(frames[k], frames[k + 1], cfg, ctx)
        assert np.abs(r.transform.rotation - one.transform.rotation).max() <= 1e-8
    for k in range(5):
        assert rotation_angle_between(traj[k].rotation, z["traj_R"][k]) <= 4e-4
        assert np.linalg.norm(traj[k].translation - z["traj_t"][k]) <= 4e-4 * ext


def test_batch_failure_in_a_later_wave(ctx):
    """A pair that fails in one wave (non-finite source) while later waves
    still run: the error names the lowest failing pair; an empty cloud is an
    argument error before any work; the context stays usable."""
    tr = _tr()
    g = load_golden("scene3k_L3")
    bad = g["src"].copy()
    bad[3, 0] = np.inf
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    srcs = [g["src"], bad, g["src"], g["src"]]
    with pytest.raises(tr.InvalidArgument, match="pair 1"):
        tr.register_batch([g["points"]] * 4, srcs, cfg, ctx, 2)
    with pytest.raises(tr.InvalidArgument, match="empty cloud"):
        tr.register_batch([g["points"], g["points"][:0]], [g["src"], g["src"]], cfg, ctx, 2)
    res = tr.register_batch([g["points"]] * 2, [g["src"]] * 2, cfg, ctx, 2)
    one = tr.register_clouds(g["points"], g["src"], cfg, ctx)
    assert all(np.array_equal(r.transform.rotation, one.transform.rotation) for r in res)
