"""Device checkpoints: the CUDA encoder / decoder against the
format restatement (oracle/checkpoint.py, data_io.cpp:444-719).

  * device save == the reference bytes of the FP32 values widened to f64;
  * device load of any reference file == hgs_scene_upload of its values
    (FP32 rounding, canonical quaternions), optimizer state included;
  * save -> load -> save is byte-identical; training resumes from the same
    state bit for bit;
  * the loader's errors match the reference's taxonomy.
"""
import numpy as np
import pytest

import oracle as O
from oracle import checkpoint as CK
from paper_2505_13215_b200 import api as A
from paper_2505_13215_b200.scene import HybridScene, ring_camera, synthetic_scene

from .test_oracle_checkpoint import canonical, random_state, scenes_identical

pytestmark = pytest.mark.gpu
FIELDS = HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS


@pytest.fixture(scope="module")
def ctx():
    c = A.Context(0)
    yield c
    c.close()


def device_state(ctx, skipped=0) -> CK.State:
    m, v, step = ctx.adam_state()
    gn4, c4, gn3, c3 = ctx.densify_stats()
    st = CK.State(ctx.download())
    st.m, st.v, st.step, st.skipped_nonfinite = m, v, step, skipped
    st.grad_norm4, st.grad_norm3, st.count4, st.count3 = gn4, gn3, c4, c3
    return st


def trained_ctx(ctx, n4=3000, n3=2000, deg=3, steps=3):
    from paper_2505_13215_b200.train import DeviceTrainer

    target = synthetic_scene(n4, n3, sh_degree=deg, seed=11)
    scene = synthetic_scene(n4, n3, sh_degree=deg, seed=12).as_float32_exact()
    scene.duration_seconds = 2.75
    cams = [ring_camera(i, 96, 72) for i in range(4)]
    tr = DeviceTrainer(ctx, scene, cams, [0.1, 0.4, 0.6, 0.9], target=target, iterations=50)
    for it in range(steps):
        tr.step([it % 4, (it + 1) % 4])
    return tr


def test_device_save_is_reference_bytes(ctx, tmp_path):
    trained_ctx(ctx)
    p = tmp_path / "dev.hgsc"
    ctx.save_checkpoint(str(p))
    scene = ctx.download()
    assert scene.duration_seconds == 2.75
    assert p.read_bytes() == CK.encode_checkpoint(scene, device_state(ctx))
    ctx.save_checkpoint(str(p), with_state=False)
    assert p.read_bytes() == CK.encode_checkpoint(scene)


@pytest.mark.parametrize("deg", [0, 1, 3])
def test_device_load_of_reference_file(ctx, tmp_path, deg):
    scene = O.Rng(300 + deg).random_scene(70, 45, deg)
    scene.tau, scene.duration_seconds, scene.extent = 0.41, 1.5, 2.2
    st = random_state(scene, deg)
    p = str(tmp_path / "ref.hgsc")
    CK.save_checkpoint(scene, st, p)
    assert ctx.load_checkpoint(p) is True
    want = canonical(scene)
    got = ctx.download()
    assert (got.n4, got.n3, got.sh_degree, got.tau, got.extent, got.duration_seconds) == \
        (want.n4, want.n3, want.sh_degree, 0.41, 2.2, 1.5)
    for f in FIELDS:
        assert np.array_equal(getattr(got, f), getattr(want, f).astype(np.float32).astype(np.float64)), f
    dst = device_state(ctx)
    assert dst.step == 1234
    for f in FIELDS:
        assert np.array_equal(getattr(dst.m, f), getattr(st.m, f).astype(np.float32).astype(np.float64)), f
        assert np.array_equal(getattr(dst.v, f), getattr(st.v, f).astype(np.float32).astype(np.float64)), f
    assert np.array_equal(dst.grad_norm4, st.grad_norm4.astype(np.float32).astype(np.float64))
    assert np.array_equal(dst.count3, st.count3) and np.array_equal(dst.count4, st.count4)
    # the skipped counter travels too: re-save and compare the OPTS scalars
    q = tmp_path / "again.hgsc"
    ctx.save_checkpoint(str(q))
    _, st2 = CK.load_checkpoint(str(q))
    assert st2.step == 1234 and st2.skipped_nonfinite == 7


def test_bare_file_zeroes_the_state(ctx, tmp_path):
    trained_ctx(ctx, steps=2)
    scene = O.Rng(5).random_scene(20, 30, 1)
    p = str(tmp_path / "bare.hgsc")
    CK.save_checkpoint(scene, None, p)
    assert ctx.load_checkpoint(p) is False
    st = device_state(ctx)
    assert st.step == 0
    assert all(not getattr(st.m, f).any() and not getattr(st.v, f).any() for f in FIELDS)
    assert not st.grad_norm4.any() and not st.count3.any()


def test_save_load_save_identical_and_resume(ctx, tmp_path):
    from paper_2505_13215_b200.train import DeviceTrainer

    tr = trained_ctx(ctx, steps=4)
    a, b = tmp_path / "a.hgsc", tmp_path / "b.hgsc"
    ctx.save_checkpoint(str(a))
    before_scene, before_state = ctx.download(), device_state(ctx)
    ctx2 = A.Context(0)
    try:
        assert ctx2.load_checkpoint(str(a))
        ctx2.save_checkpoint(str(b))
        assert a.read_bytes() == b.read_bytes()
        assert scenes_identical(ctx2.download(), before_scene)
        st2 = device_state(ctx2)
        assert st2.step == before_state.step
        # resume: the same next iteration on both contexts (gradient
        # accumulation order may differ: FP32 tolerance)
        tr2 = DeviceTrainer.__new__(DeviceTrainer)
        tr2.__dict__.update(tr.__dict__)
        tr2.ctx = ctx2
        tr.iter = tr2.iter = 4
        l1 = tr.step([1, 2])
        l2 = tr2.step([1, 2])
        assert l1 == pytest.approx(l2, rel=1e-6)
        s1, s2 = ctx.download(), ctx2.download()
        for f in FIELDS:
            np.testing.assert_allclose(getattr(s2, f), getattr(s1, f), rtol=1e-4, atol=1e-6)
    finally:
        ctx2.close()


def test_device_load_errors(ctx, tmp_path):
    scene = O.Rng(102).random_scene(8, 8)
    good = CK.encode_checkpoint(scene)
    p = tmp_path / "x.hgsc"

    def load(b):
        p.write_bytes(bytes(b))
        return ctx.load_checkpoint(str(p))

    bad = bytearray(good)
    bad[len(bad) // 2] ^= 1
    with pytest.raises(A.IntegrityError):
        load(bad)
    for keep in (len(good) - 1, len(good) // 2, 10):
        with pytest.raises(A.FormatError):
            load(good[:keep])
    bad = bytearray(good)
    bad[4] = 99
    with pytest.raises(A.UnsupportedVersionError):
        load(bad)
    with pytest.raises(A.FormatError):
        ctx.load_checkpoint(str(tmp_path / "missing.hgsc"))
    s2 = scene.copy()
    s2.quat3[3] = [0.5, 0.5, 0.5, 0.6]
    with pytest.raises(A.FormatError, match="non-unit"):
        load(CK.encode_checkpoint(s2))
    assert ctx.counts() == (0, 0)  # a rejected decode leaves an empty scene
    # the context stays usable
    assert load(good) is False
    got = ctx.download()
    for f in FIELDS:
        assert np.array_equal(getattr(got, f), getattr(canonical(scene), f).astype(np.float32).astype(np.float64))


def test_checkpoint_of_larger_scene_renders_identically(ctx, tmp_path):
    scene = synthetic_scene(60000, 40000, sh_degree=3, seed=21).as_float32_exact()
    ctx.upload(scene)
    cam = ring_camera(1, 320, 240)
    img = ctx.render(cam, 0.3)["rgb"]
    p = str(tmp_path / "big.hgsc")
    ctx.save_checkpoint(p, with_state=False)
    A.save_checkpoint(scene, str(tmp_path / "host.hgsc"))
    assert open(p, "rb").read() == open(str(tmp_path / "host.hgsc"), "rb").read()
    ctx.upload(HybridScene())
    ctx.load_checkpoint(p)
    assert np.array_equal(ctx.render(cam, 0.3)["rgb"], img)


def test_device_load_of_golden_file(ctx, tmp_path):
    """tests/golden/ckpt_small.hgsc (frozen bytes) through the CUDA decoder."""
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ckpt_small.hgsc")
    ref_scene, ref_state = CK.decode_checkpoint(open(path, "rb").read())
    assert ctx.load_checkpoint(path) is True
    got, st = ctx.download(), device_state(ctx)
    for f in FIELDS:
        assert np.array_equal(getattr(got, f), getattr(ref_scene, f).astype(np.float32).astype(np.float64)), f
        assert np.array_equal(getattr(st.m, f), getattr(ref_state.m, f).astype(np.float32).astype(np.float64)), f
    assert st.step == 321
    q = tmp_path / "re.hgsc"
    ctx.save_checkpoint(str(q))
    _, st2 = CK.load_checkpoint(str(q))
    assert st2.skipped_nonfinite == 4 and np.array_equal(st2.count3, ref_state.count3)
