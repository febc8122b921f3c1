"""Device numerics are the oracle's numerics: the Jacobi eigensolvers of
trg_math.cuh give BIT-IDENTICAL results to the CPU restatement (and thus to
the reference build) for the same inputs (-fmad=false, IEEE sqrt/div)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev_eig(ctx, n, mats):
    from paper_1807_02587_b200 import _lib
    k = 6 if n == 6 else 3
    mats = np.ascontiguousarray(mats, dtype=np.float64)
    cnt = len(mats)
    ev, vec, st = np.zeros((cnt, k)), np.zeros((cnt, k, k)), np.zeros(cnt, np.int32)
    rc = _lib.lib().trg_debug_eig(ctx.h, n, mats.ctypes.data_as(_lib.dp), cnt,
                                  ev.ctypes.data_as(_lib.dp), vec.ctypes.data_as(_lib.dp),
                                  st.ctypes.data_as(_lib.ip))
    assert rc == 0
    return ev, vec, st


def _spd(rng, cnt, k):
    out = []
    for _ in range(cnt):
        a = rng.standard_normal((k, k))
        q, _ = np.linalg.qr(a)
        lam = 10.0 ** rng.uniform(-6, 1, k)
        out.append(q @ np.diag(lam) @ q.T)
    return np.array(out)


def test_eig_sym3_bit_identical_to_oracle(ctx, port):
    rng = np.random.default_rng(0)
    mats = _spd(rng, 200, 3)
    mats[:10] = np.eye(3)  # ties
    mats[10:20] = np.diag([2.0, 5.0, 3.0])
    ev, vec, st = _dev_eig(ctx, 3, mats)
    for i, m in enumerate(mats):
        lam, ax = port.eig_sym3(m)
        assert st[i] == 0
        assert np.array_equal(lam, ev[i]) and np.array_equal(ax, vec[i]), i
    evf, vecf, _ = _dev_eig(ctx, -3, mats)
    for i, m in enumerate(mats):
        lam, ax = port.eig_sym3(m, floored=True, floor_value=1e-4)
        assert np.array_equal(lam, evf[i]) and np.array_equal(ax, vecf[i]), i


def test_jacobi6_matches_numpy(ctx):
    rng = np.random.default_rng(1)
    mats = _spd(rng, 100, 6)
    ev, vec, _ = _dev_eig(ctx, 6, mats)
    for i, m in enumerate(mats):
        ref = np.linalg.eigvalsh(m)
        assert np.allclose(ev[i], ref, rtol=1e-12, atol=1e-12 * ref.max()), (ev[i], ref)
