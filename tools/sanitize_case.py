"""Small end-to-end case for compute-sanitizer runs (one tool per run):
build + calibrate + register a 2,000-point golden pair (L = 2) and a 4,000-point
Kinect subsample (L = 3) through the C-ABI."""
import sys
sys.path.insert(0, ".")
from tests.helpers import load_golden  # noqa: E402
from paper_1807_02587_b200 import treereg as tr  # noqa: E402

ctx = tr.Context(0)
for name, L in (("lumpy2k_L2", 2), ("kinect4k_L3", 3)):
    g = load_golden(name)
    res = tr.register_clouds(g["points"], g["src"], tr.RegistrationConfig(variant=tr.Variant("adaptive", L)), ctx)
    print(name, "iterations", res.iterations, "converged", res.converged)
