"""The oracle pinned against the REFERENCE itself (CPU).

oracle/_ref/libhgs_ref.so is /root/reference/proj/src compiled from its own
sources against self-written Eigen / doctest stand-ins (oracle/ref_shim,
oracle/Makefile target ``ref``), behind a C ABI in the oracle's struct types
(oracle/ref_capi.cpp).  On the oracle's fixtures the two must agree: images,
transmittance and count maps, RenderStats and every projected splat bit for
bit; gradients, Adam updates and the conversion sweep to summation-order
rounding.  The reference's own doctest suites (proj/tests) must pass against
the same build.  Skipped only where the reference sources were never
compiled (oracle/_ref absent); tests/test_golden_cpu.py then checks the
oracle against the committed outputs of this build.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from oracle import ref as R
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference here)")

BG = (0.1, 0.2, 0.3)


def _cases():
    for seed, n3, n4, deg, (w, h) in [(201, 3, 3, 1, (32, 32)), (202, 40, 40, 3, (96, 80)), (203, 60, 20, 2, (64, 48)),
                                      (204, 0, 50, 3, (80, 64)), (205, 50, 0, 1, (80, 64))]:
        r = O.Rng(seed)
        yield r.random_scene(n3, n4, deg).as_float32_exact(), r.random_camera(w, h), 0.2 + 0.1 * (seed % 5)


@pytest.mark.parametrize("i", range(5))
def test_rasterize_bit_exact(i):
    scene, cam, t = list(_cases())[i]
    a = O.rasterize(scene, cam, t, BG, count_map=True, transmittance_map=True)
    b = R.rasterize(scene, cam, t, BG, count_map=True, transmittance_map=True)
    assert np.array_equal(a["rgb"], b["rgb"])
    assert np.array_equal(a["counts"], b["counts"])
    assert np.array_equal(a["transmittance"], b["transmittance"])
    assert a["stats"] == b["stats"]


def test_rasterize_c1_like_bit_exact_threads():
    """A 20k-Gaussian c1-shaped scene (SURVEY.md 8d generator) at 320x240,
    tile threads on both sides (raster.cpp:150-163)."""
    scene = synthetic_scene(20000, 0, 3, seed=1)
    cam = ring_camera(1, 320, 240)
    a = O.rasterize(scene, cam, 0.5, (0.2, 0.2, 0.2), num_threads=8)
    b = R.rasterize(scene, cam, 0.5, (0.2, 0.2, 0.2), num_threads=4)
    assert np.array_equal(a["rgb"], b["rgb"])
    assert a["stats"] == b["stats"]


@pytest.mark.parametrize("i", range(5))
def test_project_scene_bit_exact(i):
    scene, cam, t = list(_cases())[i]
    sa, sta = O.project_scene(scene, cam, t)
    sb, stb = R.project_scene(scene, cam, t)
    assert sta == stb and len(sa) == len(sb)
    for f in ("sx", "sy", "conic", "depth", "rgb", "alpha", "radius", "pool", "index", "gid", "x0", "x1", "y0", "y1",
              "depth_bits"):
        assert np.array_equal(sa[f], sb[f]), f


@pytest.mark.parametrize("i", range(5))
def test_forward_train_and_backward(i):
    """forward_train bit-exact (it equals rasterize, test_backward.cpp:98-100);
    gradients to summation order (the oracle walks pixels tile by tile)."""
    scene, cam, t = list(_cases())[i]
    w = np.random.default_rng(i).uniform(-1, 1, (cam.height, cam.width, 3))
    img, tape = O.forward_train(scene, cam, t, BG)
    ga = O.backward(scene, cam, tape, w)
    img_r, gb = R.forward_backward(scene, cam, t, BG, w)
    assert np.array_equal(img, img_r)
    for k in ga:
        a, b = np.asarray(ga[k]), np.asarray(gb[k])
        scale = max(np.abs(b).max(initial=0.0), 1e-300)
        assert np.abs(a - b).max(initial=0.0) <= 1e-12 * scale, k


def test_backward_skips_pixels_whose_gradient_is_zero_by_eigen_isZero():
    """backward.cpp:189 skips gpix.isZero(): every |component| <= 1e-12."""
    scene, cam, t = list(_cases())[1]
    w = np.random.default_rng(9).uniform(-1, 1, (cam.height, cam.width, 3))
    w[::3, ::2] *= 1e-12  # below the threshold in all three channels
    w[1::5, ::3, 1] = 2e-12  # one channel above it
    _, tape = O.forward_train(scene, cam, t, BG)
    ga = O.backward(scene, cam, tape, w)
    _, gb = R.forward_backward(scene, cam, t, BG, w)
    for k in ga:
        a, b = np.asarray(ga[k]), np.asarray(gb[k])
        assert np.abs(a - b).max(initial=0.0) <= 1e-12 * max(np.abs(b).max(initial=0.0), 1e-300), k


def test_photometric_loss_with_grad():
    g = np.random.default_rng(3)
    for (h, w) in [(16, 16), (37, 53)]:
        a, b = g.uniform(size=(h, w, 3)), g.uniform(size=(h, w, 3))
        for lam in (0.0, 0.2, 1.0):
            la, ga = O.photometric_loss_with_grad(a, b, lam)
            lb, gb = R.photometric_loss_with_grad(a, b, lam)
            assert la == pytest.approx(lb, rel=1e-14, abs=1e-300)
            assert np.abs(ga - gb).max() <= 1e-14 * np.abs(gb).max()


def test_sweep_convert():
    """scene.cpp:43-71: the same moved list and pools (the polar factor
    through each side's SVD agrees to rounding)."""
    scene = O.Rng(33).random_scene(7, 200, 2).as_float32_exact()
    scene.tau = 0.3
    ref_out, ref_moved, ref_rep = R.sweep_convert(scene)
    mine = scene.copy()
    moved, rep = O.sweep_convert(mine, None)
    assert np.array_equal(moved, ref_moved) and rep["count"] == ref_rep["count"] > 0
    assert (mine.n4, mine.n3) == (ref_out.n4, ref_out.n3)
    assert rep["max_leakage"] == pytest.approx(ref_rep["max_leakage"], rel=1e-12)
    for f in ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4", "mean3", "log_s3", "sh3"):
        assert np.array_equal(getattr(mine, f), getattr(ref_out, f)), f
    assert np.abs(mine.quat3 - ref_out.quat3).max() <= 1e-14
    assert np.abs(mine.op3 - ref_out.op3).max() <= 1e-13


def test_optimizer_step():
    """Three optimizer_step calls (train.cpp:131-180) from fresh state."""
    r = O.Rng(91)
    scene = r.random_scene(30, 30, 1).as_float32_exact()
    cam = r.random_camera(64, 64)
    _, tape = O.forward_train(scene, cam, 0.5, BG)
    g = O.backward(scene, cam, tape, np.random.default_rng(0).uniform(-1, 1, (64, 64, 3)))
    g["mean3"][3, 1] = np.nan  # a skipped row
    ref_scene, ref_skipped = R.optimizer_steps(scene, g, 3, mean_lr_scale=0.7)
    mine = scene.copy()
    st = O.AdamState(mine)
    for _ in range(3):
        O.optimizer_step(mine, g, st, mean_lr_scale=0.7)
    assert st.skipped_nonfinite == ref_skipped == 3
    for f in ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4", "mean3", "quat3", "log_s3", "op3", "sh3"):
        assert np.array_equal(getattr(mine, f), getattr(ref_scene, f)), f


def test_unit_quaternion_constructor_path():
    """The reference building its quaternions through UnitQuat's constructor
    (which renormalises, gauss_math.cpp:27-33): for quaternions unit in FP64
    the result is the oracle's up to the last-ulp change of the division;
    for FP32-rounded ones (|q| = 1 +- 6e-8) it moves the image by ~1e-8."""
    r = O.Rng(207)
    scene = r.random_scene(30, 30, 3)
    cam = r.random_camera(80, 64)
    R.lib().hgsr_set_quat_ctor(1)
    try:
        b = R.rasterize(scene, cam, 0.5, BG)
        b32 = R.rasterize(scene.as_float32_exact(), cam, 0.5, BG)
    finally:
        R.lib().hgsr_set_quat_ctor(0)
    a = O.rasterize(scene, cam, 0.5, BG)
    a32 = O.rasterize(scene.as_float32_exact(), cam, 0.5, BG)
    assert np.abs(a["rgb"] - b["rgb"]).max() <= 1e-14 and a["stats"] == b["stats"]
    assert np.abs(a32["rgb"] - b32["rgb"]).max() <= 1e-6 and a32["stats"] == b32["stats"]


def test_reference_doctest_suites_pass():
    """proj/tests/test_*.cpp (70 test cases) against the shim build."""
    exe = os.path.join(os.path.dirname(R.LIB_PATH), "ref_tests")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "failed: 0" in out.stdout
