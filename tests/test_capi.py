"""The product C-ABI library loads and exports every symbol that
include/treereg_b200.h declares; without a GPU it fails loudly (CPU only)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="treereg_b200.h"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(trg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("trg_build_tree", "trg_associate", "trg_solve_mstep", "trg_register_with_tree",
              "trg_register_clouds", "trg_tree_upload", "trg_ctx_create"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1807_02587_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_host_library_exports_its_header():
    """libtrg_host.so (ingest + synthetic inputs, no device code) exports
    exactly include/treereg_b200_host.h; the product library does not carry
    those host ports."""
    from paper_1807_02587_b200 import _lib
    H = ctypes.CDLL(_lib.HOST_LIB_PATH)
    host = declared_symbols("treereg_b200_host.h")
    assert host and not [s for s in host if not hasattr(H, s)]
    assert set(host) == set(_lib.HOST_SIGNATURES)
    P = ctypes.CDLL(_lib.LIB_PATH)
    assert not [s for s in host if s != "trg_host_last_error" and hasattr(P, s)]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1807_02587_b200 import treereg
    with pytest.raises(treereg.CudaError):
        treereg.Context(0)
