"""hgs_render_sweep (config c5's render sweep over t): capacity-mode renders
without host round trips give exactly the images and RenderStats of
per-frame hgs_render calls, including frames that overflow the learned
instance capacity (re-rendered exactly before the call returns)."""
import numpy as np
import pytest

from paper_2505_13215_b200 import api as A
from paper_2505_13215_b200.scene import Camera, ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = A.Context(0)
    yield c
    c.close()


def per_frame(ctx, cams, ts, bg, fixups=None):
    imgs, stats = [], []
    for c, t in zip(cams, ts):
        o = ctx.render(c, t, bg)
        imgs.append(o["rgb"])
        stats.append(o["stats"])
        if fixups is not None:
            fixups.append(ctx.render_info()["fixup_pixels"])
    return np.stack(imgs), stats


def test_sweep_equals_per_frame_renders(ctx):
    scene = synthetic_scene(40000, 20000, sh_degree=3, seed=8).as_float32_exact()
    ctx.upload(scene)
    cams = [ring_camera(8, 320, 240, index=i % 6, n_ring=6) for i in range(12)]
    ts = [j / 11.0 for j in range(12)]
    bg = (0.2, 0.3, 0.4)
    fixups = []
    ref, ref_stats = per_frame(ctx, cams, ts, bg, fixups)
    # FP64 fix-up pixels in the frames whose tape the sweep does not keep: their
    # walks read the records through the depth order (remap) -- exercised here
    assert sum(fixups[:-1]) > 0, fixups
    got, stats = ctx.render_sweep(cams, ts, bg, out="host", with_stats=True)
    assert np.array_equal(got, ref)
    assert stats == ref_stats
    got2 = ctx.render_sweep(cams, ts, bg, out="host")  # learned capacity, no first synchronous frame
    assert np.array_equal(got2, ref)


def test_sweep_capacity_overflow_is_redone(ctx):
    scene = synthetic_scene(40000, 20000, sh_degree=2, seed=9).as_float32_exact()
    ctx.upload(scene)  # resets the learned capacity
    away = Camera.look_at([0, 0, -40], [0, 0, -80], [0, -1, 0], 300.0, 320, 240)  # sees (almost) nothing
    cams = [away] + [ring_camera(9, 320, 240, index=i, n_ring=5) for i in range(5)]
    ts = [0.5] * 6
    before = ctx.render_info()["sweep_redone_frames"]
    ref, _ = per_frame(ctx, cams, ts, (0, 0, 0))
    got = ctx.render_sweep(cams, ts, (0, 0, 0), out="host")
    assert np.array_equal(got, ref)
    assert ctx.render_info()["sweep_redone_frames"] > before
    # the grown capacity holds now
    mid = ctx.render_info()["sweep_redone_frames"]
    got = ctx.render_sweep(cams[1:], ts[1:], (0, 0, 0), out="host")
    assert np.array_equal(got, ref[1:])
    assert ctx.render_info()["sweep_redone_frames"] == mid


def test_sweep_device_output_and_errors(ctx):
    import torch

    scene = synthetic_scene(20000, 10000, sh_degree=1, seed=10).as_float32_exact()
    ctx.upload(scene)
    cams = [ring_camera(10, 160, 120, index=i, n_ring=4) for i in range(4)]
    ts = [0.1, 0.4, 0.6, 0.9]
    ref, _ = per_frame(ctx, cams, ts, (0, 0, 0))
    out = torch.zeros((4, 120, 160, 3), dtype=torch.float32, device="cuda")
    ctx.render_sweep(cams, ts, (0, 0, 0), out=out)
    assert np.array_equal(out.cpu().numpy(), ref)
    with pytest.raises(ValueError):
        ctx.render_sweep(cams + [ring_camera(10, 80, 60)], ts + [0.5], (0, 0, 0), out="host")
    bad = scene.copy()
    bad.quat3[5] = [2.0, 0.0, 0.0, 0.0]
    ctx.upload(bad)
    with pytest.raises(ValueError, match="quaternion"):
        ctx.render_sweep(cams, ts, (0, 0, 0))


def test_sweep_overflow_inside_the_last_duplication_block(ctx):
    """A capacity that is not a multiple of the 1024-instance duplication
    block, overflowed by a frame whose instances still fit in that last block
    (capacity < I <= blocks * 1024): the last block must bound its splat range
    by its nominal end -- the frame is flagged, redone exactly."""
    scene = synthetic_scene(30000, 10000, sh_degree=1, seed=12).as_float32_exact()
    ctx.upload(scene)
    cam = ring_camera(12, 320, 240, index=2, n_ring=6)
    ref, _ = per_frame(ctx, [cam], [0.5], (0, 0, 0))
    ctx.render(cam, 0.5, (0, 0, 0))
    n_inst = ctx.render_info()["instances"]
    cap = n_inst - 1
    if cap % 1024 == 0:
        cap -= 1
    assert cap % 1024 != 0 and -(-cap // 1024) * 1024 >= n_inst > cap
    before = ctx.render_info()["sweep_redone_frames"]
    for _ in range(3):
        ctx._check(ctx._lib.hgs_debug_set_sweep_capacity(ctx.handle, cap))
        got = ctx.render_sweep([cam, cam], [0.5, 0.5], (0, 0, 0), out="host")
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[0])
    assert ctx.render_info()["sweep_redone_frames"] >= before + 3


def test_repeated_sweeps_are_bit_identical(ctx):
    """The fused duplication (decoupled look-back across CTAs) and the
    atomics-free forward give the same bits on every run: 40 frames of one
    view in one sweep, twice, against one per-frame render."""
    scene = synthetic_scene(100000, 0, sh_degree=3, seed=1).as_float32_exact()
    ctx.upload(scene)
    cam = ring_camera(1, 640, 480, index=0, n_ring=16)
    ref, ref_stats = per_frame(ctx, [cam], [0.5], (0.2, 0.2, 0.2))
    for _ in range(2):
        got, stats = ctx.render_sweep([cam] * 40, [0.5] * 40, (0.2, 0.2, 0.2), out="host", with_stats=True)
        assert all(np.array_equal(g, ref[0]) for g in got)
        assert all(s == ref_stats[0] for s in stats)


@pytest.mark.parametrize("overflow", [False, True])
def test_backward_after_a_sweep_uses_the_last_frame(ctx, overflow):
    """A sweep keeps only the last frame's tape (the earlier frames skip the
    backward-only outputs: the gid -> sorted map, the depth-ordered records,
    K1's SH Jacobian): hgs_backward right after the sweep gives the gradients
    of a plain render of that frame -- also when capacity overflows made
    the sweep re-render frames."""
    scene = synthetic_scene(20000, 10000, sh_degree=2, seed=18).as_float32_exact()
    ctx.upload(scene)
    cams = [ring_camera(18, 160, 120, index=i % 5, n_ring=5) for i in range(5)]
    ts = [0.1, 0.3, 0.5, 0.7, 0.9]
    bg = (0.2, 0.2, 0.2)
    w = np.random.default_rng(18).uniform(-1, 1, (120, 160, 3))
    ctx.forward_train(cams[-1], ts[-1], bg)
    ctx.zero_grads()
    ctx.backward(w)
    ref = ctx.grads()
    ctx.render(cams[0], ts[0], bg)  # a different frame's tape, so stale state would show
    if overflow:
        ctx._check(ctx._lib.hgs_debug_set_sweep_capacity(ctx.handle, 1024))  # every frame overflows: redone
    ctx.render_sweep(cams, ts, bg)
    ctx.zero_grads()
    ctx.backward(w)
    got = ctx.grads()
    for f in ("mean_x", "mean_t", "ql", "log_s4", "op4", "sh4", "mean3", "quat3", "op3", "sh3"):
        a, b = np.asarray(got[f]), np.asarray(ref[f])
        assert np.allclose(a, b, rtol=1e-5, atol=1e-7 * max(1e-30, np.abs(b).max())), f
