"""B200-native HGMR hot path (Eckart et al., arXiv 1807.02587).

``treereg`` mirrors the reference's C++ API (namespace treereg) over the
C-ABI of ``libtrg_cuda.so`` (include/treereg_b200.h).
"""
from . import treereg  # noqa: F401
