"""Device frame rendering of the synthetic C2 / C3 / C5 inputs (SURVEY 8f
rank 3): the Kinect / LiDAR pairs cast on the GPU (trg_render_*_frames) from
the host generator's poses and noise draws must equal the host generator's
frames BIT FOR BIT (one ray-casting source, trg_raycast.h, IEEE operations in
the same order on both sides)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tr():
    from paper_1807_02587_b200 import treereg
    return treereg


@pytest.mark.parametrize("seed", [2, 7, 1234])
def test_kinect_pair_device_bitwise(ctx, seed):
    tr = _tr()
    tg, sr, gt = tr.kinect_pair(seed)
    dtg, dsr, dgt = tr.kinect_pair_device(seed, ctx)
    assert np.array_equal(dtg.cpu().numpy(), tg)
    assert np.array_equal(dsr.cpu().numpy(), sr)
    assert np.array_equal(dgt.rotation, gt.rotation) and np.array_equal(dgt.translation, gt.translation)


@pytest.mark.parametrize("seed", [3, 11])
def test_lidar_pair_device_bitwise(ctx, seed):
    tr = _tr()
    tg, sr, gt = tr.lidar_pair(seed)
    dtg, dsr, dgt = tr.lidar_pair_device(seed, ctx)
    assert np.array_equal(dtg.cpu().numpy(), tg)
    assert np.array_equal(dsr.cpu().numpy(), sr)
    assert np.array_equal(dgt.rotation, gt.rotation)


def test_device_frames_register_like_host_frames(ctx):
    """The device-rendered C2 pair registers to the same bits as the host pair."""
    tr = _tr()
    cfg = tr.RegistrationConfig(variant=tr.Variant("adaptive", 3))
    tg, sr, _ = tr.kinect_pair(5)
    dtg, dsr, _ = tr.kinect_pair_device(5, ctx)
    a = tr.register_clouds(tg, sr, cfg, ctx)
    b = tr.register_clouds(dtg, dsr, cfg, ctx)
    assert np.array_equal(a.transform.rotation, b.transform.rotation)
    assert a.iterations == b.iterations


def test_render_errors(ctx):
    tr = _tr()
    from paper_1807_02587_b200 import _lib
    import ctypes as C
    R = np.eye(3)
    assert _lib.lib().trg_render_kinect_frames(ctx.h, 0, R.ctypes.data_as(_lib.dp), R.ctypes.data_as(_lib.dp),
                                               None, 1.0, C.c_void_p(0)) == _lib.TRG_EINVAL
