"""ICP point-to-point comparator on the GPU vs the
reference's register_clouds variant icp (tests/golden/make_golden_icp.py):
exact nearest neighbours (ties to the lowest index, like KdTree3), Kabsch
update, the reference's convergence test.  Bars as north_star."""
import glob
import os

import numpy as np
import pytest

from tests.helpers import GOLDEN, rotation_angle_between

pytestmark = pytest.mark.gpu

NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "icp_*.npz")))


@pytest.mark.parametrize("name", NAMES)
def test_icp_matches_reference(ctx, name):
    from paper_1807_02587_b200 import treereg as tr
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = tr.RegistrationConfig(variant=tr.Variant.parse("icp"))
    res = tr.register_clouds(z["points"], z["src"], cfg, ctx)
    ext = float(np.linalg.norm(z["points"].max(0) - z["points"].min(0)))
    assert rotation_angle_between(res.transform.rotation, z["rc_R"]) <= 1e-4
    assert np.linalg.norm(res.transform.translation - z["rc_t"]) <= 1e-4 * ext
    assert res.iterations == int(z["rc_meta"][0])
    assert res.converged == bool(z["rc_meta"][1])
    assert (res.eval_counts == 0).all() and res.model_components == len(z["points"])
    assert (np.diff(res.criterion_trace) <= 1e-12).all()  # ICP never increases the error
