"""K8 + the device EM loop vs the reference (golden fixtures from the
reference build): solve_mstep on the reference's own moments, and
register_with_tree end to end.  Tolerances: transforms 1e-4 rad and
1e-4 x scene extent (north_star); we also record the much tighter
agreement actually reached."""
import numpy as np
import pytest

from tests.helpers import golden_names, load_golden, rel_err, rotation_angle_between

pytestmark = pytest.mark.gpu


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


@pytest.mark.parametrize("name", golden_names())
def test_solve_mstep_matches_reference(ctx, name):
    tr = _tr()
    g = load_golden(name)
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    ms = tr.MomentSet(g["lc001_m0"], g["lc001_m1"], None, int(g["lc001_counts"][0]))
    sol = tr.solve_mstep(tr.make_virtual_points(ms, tree))
    assert sol.n_virtual_points == int(g["solve_scalars"][3])
    assert np.abs(sol.omega - g["solve_omega"]).max() <= 1e-9
    assert np.abs(sol.translation - g["solve_translation"]).max() <= 1e-9
    assert rel_err(sol.criterion_before, g["solve_scalars"][0]) <= 1e-10
    assert rel_err(sol.condition_estimate, g["solve_scalars"][2]) <= 1e-8
    assert abs(sol.criterion_after - g["solve_scalars"][1]) <= 1e-8 * max(1.0, g["solve_scalars"][0])
    assert np.abs(sol.delta.rotation - g["solve_R"]).max() <= 1e-9


@pytest.mark.parametrize("name", golden_names())
def test_make_virtual_points_on_device(ctx, name):
    """make_virtual_points (mstep.cpp:8-30) on the GPU: the order-preserving
    m0 > 1e-8 N filter, pi* = m0 / N and mu* = m1 / m0 (IEEE divisions:
    bit-exact)."""
    tr = _tr()
    g = load_golden(name)
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    N = int(g["lc001_counts"][0])
    m0, m1 = np.asarray(g["lc001_m0"]), np.asarray(g["lc001_m1"]).reshape(-1, 3)
    vps = tr.make_virtual_points(tr.MomentSet(m0, m1, None, N), tree)
    keep = np.nonzero(m0 > 1e-8 * N)[0]
    assert np.array_equal(vps.index, keep)
    assert np.array_equal(vps.pi_star, m0[keep] / N)
    assert np.array_equal(vps.mu_star, m1[keep] / m0[keep][:, None])
    assert vps.size() == int(g["solve_scalars"][3])


def test_solve_mstep_degenerate(ctx):
    tr = _tr()
    g = load_golden("blobs1k_L2")
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    m0 = np.zeros(tree.size())
    m1 = np.zeros((tree.size(), 3))
    m0[:2] = 10.0
    m1[:2] = g["tree"]["mean"][:2] * 10.0
    with pytest.raises(tr.DegenerateGeometryError):
        tr.solve_mstep(tr.make_virtual_points(tr.MomentSet(m0, m1, None, 100), tree))
    with pytest.raises(tr.InvalidArgument):
        tr.make_virtual_points(tr.MomentSet(m0, m1, None, 0), tree)


@pytest.mark.parametrize("name", golden_names())
def test_register_with_tree_matches_reference(ctx, name):
    tr = _tr()
    g = load_golden(name)
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    diag = float(g["reg_meta"][2])
    res = tr.register_with_tree(tree, g["src"], tr.RegistrationConfig(), diag)
    ang = rotation_angle_between(res.transform.rotation, g["reg_R"])
    dt = np.linalg.norm(res.transform.translation - g["reg_t"])
    assert ang <= 1e-4, ang
    assert dt <= 1e-4 * diag, dt
    assert res.converged == bool(g["reg_meta"][1])
    assert abs(res.iterations - int(g["reg_meta"][0])) <= 1
    n = min(res.iterations, len(g["reg_crit_before"]))
    assert rel_err(res.criterion_trace[:n], g["reg_crit_before"][:n]) <= 1e-6
    # tighter than the contract in practice:
    assert ang <= 1e-6 and dt <= 1e-6 * diag


def test_register_self_is_fixed_point(ctx):
    tr = _tr()
    g = load_golden("lumpy2k_L2")
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    res = tr.register_with_tree(tree, g["points"], tr.RegistrationConfig(), 1.0)
    assert res.converged and res.iterations <= 3
    assert np.degrees(res.transform.rotation_angle()) < 1e-2


def test_register_rejects_bad_source(ctx):
    tr = _tr()
    g = load_golden("lumpy2k_L2")
    tree = tr.GmmTree.from_host(g["tree"], ctx)
    bad = g["points"].copy()
    bad[5, 1] = np.nan
    with pytest.raises(tr.InvalidArgument):
        tr.register_with_tree(tree, bad)
    with pytest.raises(tr.InvalidArgument):
        tr.register_with_tree(tree, np.zeros((0, 3)))
