"""Host-side generators of the product library reproduce the reference's
generators bit for bit (CPU only; no GPU needed for these entry points)."""
import numpy as np
import pytest

from tests.helpers import load_golden


def _lib():
    from paper_1807_02587_b200 import treereg
    return treereg


@pytest.mark.parametrize("kind,n,seed", [("lumpy", 3000, 1), ("scene", 5000, 4),
                                         ("blobs", 1001, 5), ("sphere", 700, 3),
                                         ("plane", 333, 2)])
def test_generators_match_reference(ref, kind, n, seed):
    assert np.array_equal(_lib().synthetic(kind, n, seed), ref.synthetic(kind, n, seed))


def test_unit_normalized_and_transform_match_reference(ref):
    tr = _lib()
    p = tr.synthetic("lumpy", 10000, 1)
    assert np.array_equal(tr.unit_normalized(p), ref.unit_normalized(p))
    assert tr.bbox_diagonal(p) == ref.bbox_diagonal(p)
    for seed in range(6):
        T = tr.random_rigid_transform(15.0, 0.05, seed)
        R, t = ref.random_rigid_transform(15.0, 0.05, seed)
        assert np.array_equal(T.rotation, R) and np.array_equal(T.translation, t)


def test_golden_inputs_reproducible():
    tr = _lib()
    g = load_golden("lumpy2k_L2")
    assert np.array_equal(tr.unit_normalized(tr.synthetic("lumpy", 2000, 1)), g["points"])


def test_kinect_and_lidar_pairs():
    tr = _lib()
    tg, sr, T = tr.kinect_pair(2)
    assert tg.shape == (76800, 3) and np.isfinite(tg).all() and np.isfinite(sr).all()
    assert 0.5 < tg[:, 2].min() and tg[:, 2].max() < 6.0
    ang = np.degrees(T.rotation_angle())
    assert 0.0 < ang < 5.0 * np.sqrt(3) + 1e-9
    tg2, _, _ = tr.kinect_pair(2)
    assert np.array_equal(tg, tg2)  # deterministic
    lt, ls, LT = tr.lidar_pair(3)
    r = np.linalg.norm(lt, axis=1)
    assert lt.shape == (72000, 3) and 2.0 < r.min() and r.max() < 62.0
    assert abs(LT.translation[0] - 1.0) < 0.1


def test_pair_plans_match_the_generators():
    """The host halves of the device frame renderer (trg_synth_*_pair_plan):
    the same ground truth as the full generators, the first pixel / beam of
    each frame re-cast on the host from the plan equal to the generator's
    (the device renderer's bit-identity is tests/test_render_gpu.py)."""
    import ctypes as C
    from paper_1807_02587_b200 import _lib as L
    tr = _lib()
    H = L.host_lib()
    d = lambda a: a.ctypes.data_as(L.dp)  # noqa: E731
    tg, sr, T = tr.kinect_pair(4)
    R, t, noise = np.zeros((2, 3, 3)), np.zeros((2, 3)), np.zeros(2 * 76800)
    Rg, tg_ = np.zeros((3, 3)), np.zeros(3)
    assert H.trg_synth_kinect_pair_plan(4, 5.0, 0.05, d(R), d(t), d(noise), d(Rg), d(tg_)) == 0
    assert np.array_equal(Rg, T.rotation) and np.array_equal(tg_, T.translation)
    assert np.isfinite(noise).all() and 0.9 < noise.std() < 1.1
    lt, ls, LT = tr.lidar_pair(3)
    R2, t2, n2, tab = np.zeros((2, 3, 3)), np.zeros((2, 3)), np.zeros(2 * 72000), np.zeros(4564)
    assert H.trg_synth_lidar_pair_plan(3, d(R2), d(t2), d(n2), d(tab), d(Rg), d(tg_)) == 0
    assert np.array_equal(Rg, LT.rotation) and np.array_equal(tg_, LT.translation)
    az = np.arange(2250) * 0.16 * 0.017453292519943295
    assert np.allclose(tab[:2250], np.cos(az), atol=1e-15) and np.allclose(tab[2250:4500], np.sin(az), atol=1e-15)
    assert H.trg_synth_kinect_pair_plan(4, 5.0, 0.05, None, d(t), d(noise), d(Rg), d(tg_)) != 0
