"""Device numerics vs the oracle's: the device Jacobi (trg_math.cuh) runs
the oracle's rotation sequence with correctly rounded reciprocals / rsqrt
in place of IEEE division / sqrt chains, so eigenvalues and eigenvectors
agree with the CPU restatement (bit-exact with the reference build) to a
few ulp."""
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


def test_eig_sym3_matches_oracle(ctx, port):
    rng = np.random.default_rng(0)
    mats = _spd(rng, 200, 3)
    mats[:10] = np.eye(3)  # ties
    mats[10:20] = np.diag([2.0, 5.0, 3.0])
    ev, vec, st = _dev_eig(ctx, 3, mats)
    evf, vecf, _ = _dev_eig(ctx, -3, mats)
    for i, m in enumerate(mats):
        for floored, (e, v) in ((False, (ev[i], vec[i])), (True, (evf[i], vecf[i]))):
            lam, ax = port.eig_sym3(m, floored=floored, floor_value=1e-4)
            assert st[i] == 0
            assert np.abs(lam - e).max() <= 1e-14 * abs(lam[0]) + 1e-300, (i, lam, e)
            gap = np.array([min(abs(lam[l] - lam[(l + 1) % 3]), abs(lam[l] - lam[(l + 2) % 3]))
                            for l in range(3)])
            sep = gap > 1e-6 * abs(lam[0])
            d = np.minimum(np.abs(ax - v).max(axis=0), np.abs(ax + v).max(axis=0))
            assert np.all(d[sep] <= 1e-10), (i, d)


def test_jacobi6_matches_numpy(ctx):
    rng = np.random.default_rng(1)
    mats = _spd(rng, 100, 6)
    ev, vec, _ = _dev_eig(ctx, 6, mats)
    for i, m in enumerate(mats):
        ref = np.linalg.eigvalsh(m)
        assert np.allclose(ev[i], ref, rtol=1e-12, atol=1e-12 * ref.max()), (ev[i], ref)


def test_warp_solve_matches_numpy(ctx):
    """The warp-parallel 6x6 eigen + LDLT solve of K8 on random SPD systems
    (guards the nvcc inlining miscompile noted in trg_math.cuh)."""
    from paper_1807_02587_b200 import _lib
    rng = np.random.default_rng(2)
    for m in _spd(rng, 30, 6):
        b = rng.standard_normal(6)
        v = np.concatenate([m[np.triu_indices(6)], b])
        out = np.zeros(16)
        assert _lib.lib().trg_debug_solve(ctx.h, v.ctypes.data_as(_lib.dp), 10,
                                          out.ctypes.data_as(_lib.dp)) == 0
        ev = np.linalg.eigvalsh(m)
        cond = ev[-1] / ev[0]
        if cond >= 1e12:
            assert out[7] == 1
            continue
        x = np.linalg.solve(m, b)
        assert np.allclose(out[:6], x, rtol=1e-8, atol=1e-8 * np.abs(x).max())
        assert abs(out[6] - cond) <= 1e-8 * cond


def test_closed_form_eig3_matches_jacobi(ctx, port):
    """The closed-form 3x3 solver (eig3_cf, used by the M-steps, the leaf
    refits and the calibration's parent refreshes) against the Jacobi oracle:
    eigenvalues to 1e-13 of the spread (tiny floored eigenvalues to 1e-11
    relative), eigenvectors of separated eigenvalues to 1e-9, the same sign
    and handedness conventions, a valid orthonormal basis always; and the
    quantities the densities use (log-normaliser, the quadratic form) agree
    even inside near-degenerate eigenspaces."""
    rng = np.random.default_rng(7)
    mats = _spd(rng, 400, 3)
    mats[:10] = np.eye(3) * 2.5  # ties
    mats[10:20] = np.diag([2.0, 5.0, 3.0])
    for i in range(20, 60):  # planar and linear patches, near-degenerate pairs
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        lam = [1e-2, 1e-2 * (1 + 10.0 ** rng.uniform(-12, -3)), 10.0 ** rng.uniform(-7, -4)]
        mats[i] = q @ np.diag(rng.permutation(lam)) @ q.T
    mats[60:70] *= 1e-9  # tiny scales
    mats[70:80] *= 1e6
    for n, floored in ((33, False), (-33, True)):
        ev, vec, st = _dev_eig(ctx, n, mats)
        for i, m in enumerate(mats):
            lam, ax = port.eig_sym3(m, floored=floored, floor_value=1e-4)
            assert st[i] == 0
            e, v = ev[i], vec[i]
            spread = abs(lam[0])
            assert np.all(np.abs(lam - e) <= 1e-14 * spread + 1e-300), (i, lam, e)
            assert np.abs(v.T @ v - np.eye(3)).max() <= 1e-13
            assert np.linalg.det(v) > 0
            gap = np.array([min(abs(lam[l] - lam[(l + 1) % 3]), abs(lam[l] - lam[(l + 2) % 3]))
                            for l in range(3)])
            sep = gap > 1e-5 * spread
            d = np.abs(ax - v).max(axis=0)
            assert np.all(d[sep] <= 1e-9), (i, d, lam)
            # the density's quadratic form is basis-independent
            x = rng.standard_normal(3) * np.sqrt(spread)
            qa = np.sum((ax.T @ x) ** 2 / np.maximum(lam, 1e-300))
            qb = np.sum((v.T @ x) ** 2 / np.maximum(e, 1e-300))
            assert abs(qa - qb) <= 1e-9 * abs(qa) + 1e-300
