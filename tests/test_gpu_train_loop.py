"""train_scene: the reference training loop (train.cpp:382-494) on the device.

Pinned pieces: the batch schedule (rng.py, tests/test_rng.py), the first
iteration's loss against the oracle on the same batch, the sweep cadence and
pool bookkeeping, the probe PSNR and NumericAbort propagation."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200.rng import MT19937_64, uniform_index
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2505_13215_b200.api import Context

    c = Context(0)
    yield c
    c.close()


def _dataset(ctx, n_cams=4, n_frames=3, W=64, H=48):
    from paper_2505_13215_b200.train import Frame, MultiViewDataset, quantize_8bit

    target = synthetic_scene(1200, 400, 1, seed=41, density_n=1500)
    cams = [ring_camera(41, W, H, index=i, n_ring=n_cams) for i in range(n_cams)]
    ctx.upload(target)
    frames = [[Frame(time=f / max(1, n_frames - 1),
                     image=quantize_8bit(ctx.render(c, f / max(1, n_frames - 1), (0.2, 0.2, 0.2))["rgb"]
                                         .astype(np.float64)))
               for f in range(n_frames)] for c in cams]
    return MultiViewDataset(cameras=cams, frames=frames, background=(0.2, 0.2, 0.2), duration_seconds=1.0)


def test_train_scene_loop(ctx):
    from paper_2505_13215_b200.train import TrainConfig, train_scene

    ds = _dataset(ctx)
    init = synthetic_scene(1200, 400, 1, seed=42, density_n=1500, tau=0.3)
    cfg = TrainConfig(iterations=40, batch_size=2, warmup_iters=10, densify_interval=10, densify_stop_iter=0,
                      tau=0.3, seed=7, sh_degree=1, probe_interval=10)
    res = train_scene(init, ds, cfg, ctx=ctx)
    log = res.log
    assert [r.iter for r in log] == list(range(1, 41))
    assert all(math.isfinite(r.loss) for r in log)
    assert np.mean([r.loss for r in log[-5:]]) < np.mean([r.loss for r in log[:5]])
    # sweeps at 10, 20, 30, 40 only; the pools shrink / grow by the moved counts
    assert all(r.conversions == 0 for r in log if r.iter % 10)
    assert sum(r.conversions for r in log) > 0
    n0 = init.n4 + init.n3
    for r in log:
        assert r.n_static + r.n_dynamic == n0
    assert log[-1].n_static == init.n3 + sum(r.conversions for r in log)
    # probe rows
    assert [r.iter for r in log if r.probe_psnr >= 0] == [10, 20, 30, 40]
    assert res.scene.n4 == log[-1].n_dynamic and res.state[2] == 40


def test_first_iteration_loss_matches_oracle(ctx):
    """Iteration 1 draws the reference's batch and its mean loss is the
    oracle's photometric loss of the oracle renders of those views."""
    from paper_2505_13215_b200.train import TrainConfig, train_scene

    ds = _dataset(ctx)
    init = synthetic_scene(1200, 400, 1, seed=43, density_n=1500).as_float32_exact()
    cfg = TrainConfig(iterations=1, batch_size=3, warmup_iters=1, densify_stop_iter=0, seed=11, sh_degree=1,
                      probe_interval=0, conversion_enabled=False)
    res = train_scene(init, ds, cfg, ctx=ctx)
    samples = [(c, f) for c in range(len(ds.frames)) for f in range(len(ds.frames[c]))]
    g = MT19937_64(cfg.seed)
    batch = [samples[uniform_index(g, 0, len(samples) - 1)] for _ in range(cfg.batch_size)]
    ref = np.mean([O.photometric_loss(O.rasterize(init, ds.cameras[c], ds.frames[c][f].time, ds.background)["rgb"],
                                      ds.frames[c][f].image, 0.2) for c, f in batch])
    assert res.log[0].loss == pytest.approx(ref, rel=1e-5)


def test_train_scene_with_densification(ctx):
    """The full loop with the densify window open (train.cpp:456-465): pools
    change size at the densify iterations only, the loss still decreases."""
    from paper_2505_13215_b200.train import TrainConfig, train_scene

    ds = _dataset(ctx)
    init = synthetic_scene(1200, 400, 1, seed=45, density_n=1500, tau=0.3)
    sizes = []
    cfg = TrainConfig(iterations=40, batch_size=2, warmup_iters=10, densify_interval=10, densify_stop_iter=30,
                      grad_threshold=1e-4, opacity_prune_eps=0.02, tau=0.3, seed=3, sh_degree=1, probe_interval=0,
                      max_gaussians=1500, opacity_reset_enabled=True, opacity_reset_interval=20)
    res = train_scene(init, ds, cfg, ctx=ctx, on_row=lambda r: sizes.append(r.n_static + r.n_dynamic))
    log = res.log
    assert all(math.isfinite(r.loss) for r in log)
    changes = [i + 1 for i in range(1, len(sizes)) if sizes[i] != sizes[i - 1]]
    assert changes and set(changes) <= {10, 20, 30, 40}, changes
    assert res.scene.n4 <= 1500 and res.scene.n3 <= 1500 + 1200
    # the opacity reset at iteration 20 (logit(0.01) cap) makes the scene translucent
    assert max(r.loss for r in log[20:]) > min(r.loss for r in log[:20])


def test_train_scene_rejects_bad_config(ctx):
    from paper_2505_13215_b200.train import TrainConfig, train_scene

    ds = _dataset(ctx, n_cams=2, n_frames=1)
    init = synthetic_scene(100, 50, 1, seed=44)
    with pytest.raises(ValueError):
        train_scene(init, ds, TrainConfig(iterations=10, warmup_iters=20), ctx=ctx)


@pytest.mark.gpu
def test_render_gt_u8_device_matches_the_host_encoding():
    """render_gt_u8_device (configs[2]'s 5400 device-resident GT frames) encodes
    the rendered frame like linear_to_srgb8 (image.cpp:15-18) on the host."""
    import numpy as np

    from paper_2505_13215_b200.api import Context
    from paper_2505_13215_b200.scene import ring_camera, synthetic_scene
    from paper_2505_13215_b200.train import linear_to_srgb8, render_gt_u8_device

    ctx = Context(0)
    try:
        target = synthetic_scene(3000, 1000, 2, seed=11)
        cams = [ring_camera(3, 160, 120, index=i, n_ring=3) for i in range(3)]
        times = [0.1, 0.5, 0.9]
        dev = render_gt_u8_device(ctx, target, cams, times, bg=(0.2, 0.2, 0.2))
        for cam, t, d in zip(cams, times, dev):
            host = linear_to_srgb8(ctx.render(cam, t, (0.2, 0.2, 0.2))["rgb"].astype(np.float64))
            diff = np.abs(d.cpu().numpy().astype(int) - host.astype(int))
            assert diff.max() <= 1 and (diff == 0).mean() >= 0.999
    finally:
        ctx.close()
