"""GPU init_scene (data_io.cpp:189-238) against the oracle's
literal O(N^2) restatement, and training from an on-disk 8-bit dataset
 through the device HGS_U8 path.

Gate: the device scene equals the oracle's FP64 scene rounded to FP32
(bit-exact; FP64 log() on the device is within 1 ulp of glibc's, which can
only matter at an FP32 rounding tie), extent identical.
"""
import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200 import api as A
from paper_2505_13215_b200.scene import HybridScene, ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu
FIELDS = HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS


@pytest.fixture(scope="module")
def ctx():
    c = A.Context(0)
    yield c
    c.close()


def check_init(ctx, pos, rgb, cfg):
    ctx.init_scene(pos, rgb, cfg)
    got = ctx.download()
    ref = O.init_scene(pos, rgb, cfg.sh_degree, cfg.tau, cfg.duration_seconds, cfg.init_temporal_scale,
                       cfg.init_opacity)
    assert (got.n4, got.n3, got.sh_degree, got.tau, got.duration_seconds) == \
        (ref.n4, 0, cfg.sh_degree, cfg.tau, cfg.duration_seconds)
    assert got.extent == ref.extent
    for f in FIELDS:
        a, b = getattr(got, f), getattr(ref, f).astype(np.float32).astype(np.float64)
        assert np.array_equal(a, b), (f, int((a != b).sum()))


@pytest.mark.parametrize("n,deg", [(4, 0), (30, 1), (257, 2), (5000, 3)])
def test_init_scene_vs_oracle(ctx, n, deg):
    rng = np.random.default_rng(n)
    pos, rgb = rng.uniform(-2, 2, (n, 3)), rng.uniform(0, 1, (n, 3))
    check_init(ctx, pos, rgb, A.InitConfig(sh_degree=deg, tau=0.4, duration_seconds=3.0))


def test_init_scene_duplicates_and_clusters(ctx):
    """ties (zero distances, repeated points) and the 1e-4 floor"""
    rng = np.random.default_rng(3)
    base = rng.uniform(-1, 1, (300, 3))
    pos = np.concatenate([base, base[:100], base[:50] + 1e-7, rng.normal(0, 1e-6, (40, 3))])
    rgb = rng.uniform(0, 1, (pos.shape[0], 3))
    check_init(ctx, pos, rgb, A.InitConfig(sh_degree=1, init_temporal_scale=0.3, init_opacity=0.25))


def test_init_scene_errors_and_module_api(ctx):
    with pytest.raises(ValueError, match="at least 4"):
        ctx.init_scene(np.zeros((3, 3)), np.zeros((3, 3)))
    from paper_2505_13215_b200.dataset import InitPoints

    rng = np.random.default_rng(1)
    pts = InitPoints(rng.uniform(-1, 1, (64, 3)), rng.uniform(0, 1, (64, 3)))
    s = A.init_scene(pts, A.InitConfig(sh_degree=2), ctx=ctx)
    assert s.n4 == 64 and s.n3 == 0 and s.sh_degree == 2
    assert ctx.counts() == (64, 0)


def test_train_from_disk_u8_matches_linear(tmp_path):
    """load_dataset -> train_scene: the 8-bit frames (decoded on the device)
    give the same first-iteration loss as the linear float frames."""
    from paper_2505_13215_b200 import dataset as D
    from paper_2505_13215_b200.train import Frame, MultiViewDataset, TrainConfig, quantize_8bit, train_scene

    target = synthetic_scene(800, 800, sh_degree=1, seed=5)
    cams = [ring_camera(i, 64, 48) for i in range(3)]
    with A.Context(0) as c:
        c.upload(target)
        frames = [[Frame(t, quantize_8bit(c.render(cam, t)["rgb"].astype(np.float64))) for t in (0.0, 0.5, 1.0)]
                  for cam in cams]
    ds = MultiViewDataset(cameras=cams, frames=frames, duration_seconds=1.0, camera_ids=[0, 1, 2])
    root = str(tmp_path / "ds")
    D.save_dataset(ds, root)
    tr8, _ = D.load_dataset(root, frames="u8", pinned=True)
    trl, _ = D.load_dataset(root, frames="linear")
    init = synthetic_scene(800, 800, sh_degree=1, seed=6).as_float32_exact()
    cfg = TrainConfig(iterations=3, batch_size=2, warmup_iters=3, probe_interval=1, densify_interval=1000,
                      conversion_enabled=False, opacity_reset_enabled=False, sh_degree=1)
    logs = []
    for d in (tr8, trl):
        with A.Context(0) as c:
            logs.append(train_scene(init, d, cfg, ctx=c).log)
    for a, b in zip(*logs):
        assert a.loss == pytest.approx(b.loss, rel=1e-5)
        assert a.probe_psnr == pytest.approx(b.probe_psnr, abs=1e-4)


def test_train_directory_end_to_end(tmp_path):
    """hybridgs.train (bindings.cpp:221-235) on a dataset directory: points ->
    GPU kNN init -> device training with densification and sweeps ->
    held-out PSNR; the loss goes down (test_train.cpp:273-307)."""
    from paper_2505_13215_b200 import dataset as D
    from paper_2505_13215_b200.train import Frame, MultiViewDataset, TrainConfig, quantize_8bit, train_directory

    target = synthetic_scene(1500, 1500, sh_degree=1, seed=15)
    cams = [ring_camera(i, 64, 48, index=i, n_ring=4) for i in range(4)]
    with A.Context(0) as c:
        c.upload(target)
        frames = [[Frame(t, quantize_8bit(c.render(cam, t)["rgb"].astype(np.float64))) for t in (0.0, 0.5, 1.0)]
                  for cam in cams]
    rng = np.random.default_rng(3)
    pts = D.InitPoints(target.mean_x[:400].copy(), rng.uniform(0, 1, (400, 3)))
    ds = MultiViewDataset(cameras=cams, frames=frames, duration_seconds=1.0, camera_ids=[0, 1, 2, 3],
                          init_points=pts)
    root = str(tmp_path / "scene")
    D.save_dataset(ds, root)
    cfg = TrainConfig(iterations=60, batch_size=2, warmup_iters=20, densify_interval=20, densify_stop_iter=40,
                      probe_interval=20, sh_degree=1)
    with A.Context(0) as c:
        scene, held_psnr = train_directory(root, held_out=3, config=cfg, ctx=c)
    assert scene.n4 + scene.n3 > 0 and held_psnr > 5.0
    with A.Context(0) as c:
        from paper_2505_13215_b200.train import train

        split, _ = D.load_dataset(root, 3)
        res = train(split, cfg, ctx=c)
    first, last = res.log[0].loss, res.log[-1].loss
    assert last < first
