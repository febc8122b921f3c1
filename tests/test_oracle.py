"""The CPU oracle is pinned: the plain-C restatement (oracle/trg_oracle.c)
must reproduce the reference build (oracle/_ref, = /root/reference sources +
test shims) BIT FOR BIT, both on the committed golden fixtures (generated
from the reference) and live on more clouds when the reference build is
present.  CPU only."""
import numpy as np
import pytest

from tests.helpers import TREE_KEYS, golden_names, load_golden


@pytest.mark.parametrize("name", golden_names())
def test_port_matches_golden_tree(port, name):
    g = load_golden(name)
    t = port.build_tree(g["points"], max_level=int(g["max_level"]))
    for k in TREE_KEYS:
        assert np.array_equal(t[k], g["tree"][k]), k
    assert t["calibration_drift"] == g["calibration_drift"]


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("tag,lc", [("lc0", 0.0), ("lc001", 0.01), ("lc13", 1.0 / 3.0)])
def test_port_matches_golden_association(port, name, tag, lc):
    g = load_golden(name)
    m, node, w = port.associate(g["tree"], g["points"], g["R"], g["t"], lc, per_point=True)
    assert np.array_equal(m.m0, g[f"{tag}_m0"])
    assert np.array_equal(m.m1, g[f"{tag}_m1"])
    assert np.array_equal(m.m2, g[f"{tag}_m2"])
    assert [m.total_points, m.outliers, m.density_evaluations] == list(g[f"{tag}_counts"])
    assert np.array_equal(node, g[f"{tag}_node"])
    assert np.array_equal(w, g[f"{tag}_w"])


@pytest.mark.parametrize("name", golden_names())
def test_port_matches_golden_solve_and_register(port, name):
    g = load_golden(name)
    m = port.associate(g["tree"], g["points"], g["R"], g["t"], 0.01)
    s = port.solve_mstep(g["tree"], m.m0, m.m1, m.total_points)
    for k in ("omega", "translation", "R", "t"):
        assert np.array_equal(s[k], g["solve_" + k]), k
    assert s["criterion_before"] == g["solve_scalars"][0]
    assert s["criterion_after"] == g["solve_scalars"][1]
    assert s["condition"] == g["solve_scalars"][2]
    r = port.register_with_tree(g["tree"], g["src"], target_diag=float(g["reg_meta"][2]))
    assert r["iterations"] == int(g["reg_meta"][0])
    assert int(r["converged"]) == int(g["reg_meta"][1])
    assert np.array_equal(r["R"], g["reg_R"]) and np.array_equal(r["t"], g["reg_t"])
    assert np.array_equal(r["criterion_before"], g["reg_crit_before"])
    assert np.array_equal(r["eval_counts"], g["reg_evals"])


LIVE = [("blobs", 3000, 9, 2), ("lumpy", 4000, 3, 3), ("scene", 2500, 8, 3), ("plane", 800, 2, 2),
        ("sphere", 1500, 4, 3), ("scene", 600, 1, 4)]


@pytest.mark.parametrize("kind,n,seed,L", LIVE)
def test_port_matches_reference_live(ref, port, kind, n, seed, L):
    pts = ref.synthetic(kind, n, seed)
    a = ref.build_tree(pts, max_level=L)
    b = port.build_tree(pts, max_level=L)
    for k in TREE_KEYS:
        assert np.array_equal(a[k], b[k]), k
    R, t = ref.random_rigid_transform(8.0, 0.03, seed)
    ra = ref.register_with_tree(a, pts @ R.T + t, variant="tree")
    rb = port.register_with_tree(a, pts @ R.T + t, variant="tree")
    assert ra["iterations"] == rb["iterations"]
    assert np.array_equal(ra["R"], rb["R"]) and np.array_equal(ra["t"], rb["t"])


def test_port_degenerate_inputs(ref, port):
    # identical points: floored, finite model (test_gmm.cpp:231-253)
    pts = np.tile(np.array([[1.0, 1.0, 1.0]]), (200, 1))
    a = ref.build_tree(pts, max_level=2)
    b = port.build_tree(pts, max_level=2)
    for k in TREE_KEYS:
        assert np.array_equal(a[k], b[k]), k
    # validation errors map to the same codes
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e1:
        ref.build_tree(np.zeros((0, 3)), max_level=2)
    with pytest.raises(OracleError) as e2:
        port.build_tree(np.zeros((0, 3)), max_level=2)
    assert e1.value.code == e2.value.code == 1


def test_reference_unit_tests_pass_against_shims():
    """The reference's own doctest suite (proj/tests) passes on the shimmed
    build, which pins the Eigen shim's numerics (charpoly eigenvalue oracle,
    LDLT optimality, ...)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref",
                       "ref_unit_tests")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_unit_tests not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
