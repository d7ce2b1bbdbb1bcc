"""GPU evaluation path against the FP64 oracle, via the C ABI.

  * density_map (raster.cpp:268-287): bit-exact counts (boxes are bit-exact);
  * psnr (metrics.cpp:91-101): |dPSNR| <= 1e-6 dB on the same FP32 image;
  * ssim: |dSSIM| <= 1e-5 (FP32 window sums on the device);
  * evaluate_views (eval.cpp:12-23): per-frame metrics within those bounds.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200.scene import HybridScene, ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu

PSNR_TOL = 1e-6
SSIM_TOL = 1e-5


@pytest.fixture(scope="module")
def ctx():
    from paper_2505_13215_b200.api import Context

    c = Context(0)
    yield c
    c.close()


def single_static_scene(opacity_logit=1.0):
    return HybridScene(mean3=np.zeros((1, 3)), quat3=np.array([[1.0, 0, 0, 0]]), log_s3=np.zeros((1, 3)),
                       op3=np.array([opacity_logit]))


def test_density_map_random_scene(ctx):
    """test_raster.cpp:185-201 on the device"""
    rng = O.Rng(45)
    scene = rng.random_scene(5, 5).as_float32_exact()
    cam = rng.random_camera(48, 48)
    ctx.upload(scene)
    counts = ctx.density_map(cam, 0.5)
    assert (counts == O.density_map(scene, cam, 0.5)).all()
    dyn = ctx.density_map(cam, 0.5, dynamics_only=True)
    assert (dyn == O.density_map(scene, cam, 0.5, dynamics_only=True)).all()
    assert (dyn <= counts).all()


def test_density_map_module_level_single_static():
    """tests/python/test_smoke.py:84-96 through hybridgs-style density_map"""
    from paper_2505_13215_b200.api import density_map

    scene = single_static_scene()
    cam = O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], 40.0, 24, 16)
    total = density_map(scene, cam, 0.5)
    dyn = density_map(scene, cam, 0.5, dynamics_only=True)
    assert total.shape == (16, 24)
    assert total.sum() > 0
    assert (dyn <= total).all() and dyn.sum() == 0
    assert (total == O.density_map(scene, cam, 0.5)).all()


@pytest.mark.parametrize("n4,n3,size,t", [(3000, 2000, (160, 120), 0.31), (20000, 20000, (640, 360), 0.7)])
def test_density_map_synthetic(ctx, n4, n3, size, t):
    scene = synthetic_scene(n4, n3, sh_degree=3, seed=7).as_float32_exact()
    cam = ring_camera(3, *size)
    ctx.upload(scene)
    for dyn in (False, True):
        got = ctx.density_map(cam, t, dynamics_only=dyn)
        ref = O.density_map(scene, cam, t, dynamics_only=dyn)
        assert got.dtype == np.uint32 and got.shape == ref.shape
        assert (got == ref).all(), int((got != ref).sum())


def test_density_map_releases_the_tape(ctx):
    from paper_2505_13215_b200.api import StateError

    scene = synthetic_scene(200, 200, sh_degree=1, seed=1).as_float32_exact()
    cam = ring_camera(0, 64, 48)
    ctx.upload(scene)
    ctx.forward_train(cam, 0.5, (0, 0, 0))
    ctx.density_map(cam, 0.5)
    with pytest.raises(StateError):
        ctx.backward(np.zeros((48, 64, 3)))


def test_image_metrics_vs_oracle(ctx):
    scene = synthetic_scene(4000, 3000, sh_degree=3, seed=3).as_float32_exact()
    cam = ring_camera(5, 128, 96)
    ctx.upload(scene)
    img = ctx.render(cam, 0.4, (0.1, 0.2, 0.3))["rgb"].astype(np.float64)
    gt = np.clip(img + np.random.default_rng(0).normal(0, 0.05, img.shape), 0, 1).astype(np.float32)
    gt64 = gt.astype(np.float64)
    for g in (gt, gt64):  # host f32 / f64 frames
        p, s = ctx.image_metrics(g)
        assert abs(p - O.psnr(img, gt64)) <= PSNR_TOL
        assert abs(s - O.ssim(img, gt64)) <= SSIM_TOL
    p, s = ctx.image_metrics(img.astype(np.float32))
    assert math.isinf(p) and abs(s - 1.0) <= SSIM_TOL


def test_image_metrics_u8_and_device_frames(ctx):
    import torch

    from paper_2505_13215_b200.train import linear_to_srgb8, srgb8_to_linear

    scene = synthetic_scene(3000, 3000, sh_degree=2, seed=4).as_float32_exact()
    cam = ring_camera(2, 96, 80)
    ctx.upload(scene)
    img = ctx.render(cam, 0.6, (0, 0, 0))["rgb"].astype(np.float64)
    noisy = np.clip(img + np.random.default_rng(1).normal(0, 0.03, img.shape), 0, 1)
    u8 = linear_to_srgb8(noisy)
    lin = srgb8_to_linear(u8)
    p, s = ctx.image_metrics(u8)
    assert abs(p - O.psnr(img, lin)) <= PSNR_TOL
    assert abs(s - O.ssim(img, lin)) <= SSIM_TOL
    d8 = torch.from_numpy(u8).cuda()
    d32 = torch.from_numpy(lin.astype(np.float32)).cuda()
    torch.cuda.synchronize()
    p8, s8 = ctx.image_metrics(gt_device_ptr=d8.data_ptr(), gt_u8=True)
    p32, s32 = ctx.image_metrics(gt_device_ptr=d32.data_ptr())
    assert abs(p8 - p) <= 1e-9 and abs(s8 - s) <= 1e-9  # FP64 atomics: order-dependent last ulp
    assert abs(p32 - p) <= PSNR_TOL and abs(s32 - s) <= SSIM_TOL


def test_module_psnr_ssim():
    """bindings.cpp:175-180 / test_smoke.py psnr, ssim"""
    from paper_2505_13215_b200.api import HgsError, psnr, ssim

    rng = np.random.default_rng(5)
    a = rng.uniform(0, 1, (40, 50, 3))
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1)
    assert math.isinf(psnr(a, a))
    assert abs(ssim(a, a) - 1.0) <= SSIM_TOL
    # the device reads FP32 copies of both images
    a32, b32 = a.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    assert abs(psnr(a, b) - O.psnr(a32, b32)) <= PSNR_TOL
    assert abs(ssim(a, b) - O.ssim(a32, b32)) <= SSIM_TOL
    assert psnr(np.zeros((8, 8, 3)), np.full((8, 8, 3), 0.1)) == pytest.approx(20.0, rel=1e-6)
    with pytest.raises((HgsError, ValueError)):
        ssim(np.zeros((8, 8, 3)), np.zeros((8, 8, 3)))  # smaller than the window
    with pytest.raises(ValueError):
        psnr(np.zeros((4, 4, 3)), np.zeros((4, 5, 3)))


def test_evaluate_views_vs_oracle(ctx):
    from paper_2505_13215_b200.train import Frame, MultiViewDataset, evaluate_views

    scene = synthetic_scene(2000, 2000, sh_degree=3, seed=9).as_float32_exact()
    cams = [ring_camera(i, 80, 64) for i in range(3)]
    rng = np.random.default_rng(2)
    frames = [[Frame(time=float(t), image=rng.uniform(0, 1, (64, 80, 3))) for t in (0.2, 0.7)] for _ in cams]
    ds = MultiViewDataset(cameras=cams, frames=frames, background=(0.5, 0.5, 0.5))
    rep = evaluate_views(scene, ds, ctx=ctx)
    assert rep.frames == 6
    i = 0
    for ci, cam in enumerate(cams):
        for fr in frames[ci]:
            img = O.rasterize(scene, cam, fr.time, ds.background, num_threads=8)["rgb"]
            gt32 = fr.image.astype(np.float32).astype(np.float64)
            # the device image is FP32 within 1e-4 of the oracle's: compare
            # against the oracle metrics with that slack
            assert abs(rep.frame_psnr[i] - O.psnr(img, gt32)) <= 1e-3
            assert abs(rep.frame_ssim[i] - O.ssim(img, gt32)) <= 1e-4
            i += 1
    assert rep.mean_psnr == pytest.approx(sum(rep.frame_psnr) / 6, rel=1e-12)
