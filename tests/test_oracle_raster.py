"""Pins the oracle renderer against the reference's test_raster.cpp / acceptance (2)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200.scene import HybridScene

LOW_PASS = 0.3


def front_camera(size=32, focal=50.0):  # test_raster.cpp:13-15
    return O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], focal, size, size)


def test_empty_scene_is_background():
    """test_raster.cpp:26-33"""
    out = O.rasterize(HybridScene(), front_camera(), 0.3, (0.1, 0.5, 0.9))
    assert (out["rgb"] == np.array([0.1, 0.5, 0.9])).all()


def test_on_axis_closed_form():
    """test_raster.cpp:35-51"""
    cam = front_camera(64, 80.0)
    sigma = 0.2
    s = O.project_3d([0, 0, 0], sigma * sigma * np.eye(3), cam)
    assert s is not None
    assert s["sx"] == pytest.approx(cam.cx, rel=1e-12)
    assert s["sy"] == pytest.approx(cam.cy, rel=1e-12)
    assert s["depth"] == pytest.approx(3.0, rel=1e-12)
    cov2 = np.linalg.inv(np.array(s["conic"]).reshape(2, 2))
    expect = (80.0 / 3.0) ** 2 * sigma * sigma + LOW_PASS
    assert cov2[0, 0] == pytest.approx(expect, rel=1e-3)
    assert cov2[1, 1] == pytest.approx(expect, rel=1e-3)
    assert abs(cov2[0, 1]) < 1e-9


def test_culling():
    """test_raster.cpp:53-64"""
    cam = front_camera()
    stats = {}
    assert O.project_3d([0, 0, -10], 0.01 * np.eye(3), cam, stats) is None
    assert stats["culled_depth"] == 1
    tight = front_camera()
    tight.far = 2.0
    assert O.project_3d([0, 0, 0], 0.01 * np.eye(3), tight, stats) is None
    assert O.project_3d([50, 0, 0], 0.01 * np.eye(3), cam, stats) is None
    assert stats["culled_offscreen"] >= 1


def test_screen_covariance_matches_fd_jacobian():
    """test_raster.cpp:66-97"""
    g = np.random.default_rng(41)
    cam = front_camera(64, 60.0)
    for _ in range(50):
        mean = np.array([0.8 * g.standard_normal(), 0.8 * g.standard_normal(), 0.5 * g.standard_normal()])
        a = 0.05 * g.standard_normal((3, 3))
        cov = a @ a.T + 1e-4 * np.eye(3)
        s = O.project_3d(mean, cov, cam)
        if s is None:
            continue
        cp = cam.rot @ mean + cam.trans

        def screen(q):
            return np.array([cam.fx * q[0] / q[2] + cam.cx, cam.fy * q[1] / q[2] + cam.cy])

        h = 1e-6
        jac = np.zeros((2, 3))
        for c in range(3):
            qp, qm = cp.copy(), cp.copy()
            qp[c] += h
            qm[c] -= h
            jac[:, c] = (screen(qp) - screen(qm)) / (2 * h)
        expect = jac @ cam.rot @ cov @ cam.rot.T @ jac.T + LOW_PASS * np.eye(2)
        got = np.linalg.inv(np.array(s["conic"]).reshape(2, 2))
        assert np.abs(got - expect).max() < 1e-6 * np.abs(expect).max()


def test_single_splat_closed_form():
    """test_raster.cpp:131-155 (known answer, 1e-12)"""
    cam = front_camera(33, 40.0)
    sc = HybridScene(sh_degree=0, mean3=np.zeros((1, 3)), quat3=np.array([[1.0, 0, 0, 0]]),
                     log_s3=np.full((1, 3), math.log(0.3)), op3=np.array([math.log(0.7 / 0.3)]),
                     sh3=((np.array([0.9, 0.1, 0.3]) - 0.5) / 0.28209479177387814).reshape(1, 1, 3))
    bg = np.array([0.0, 0.0, 1.0])
    out = O.rasterize(sc, cam, 0.0, bg)["rgb"]
    cov = O.build_cov3(np.eye(3), [math.log(0.3)] * 3)
    s = O.project_3d([0, 0, 0], cov, cam)
    d = np.array([16.5, 16.5]) - np.array([s["sx"], s["sy"]])
    conic = np.array(s["conic"]).reshape(2, 2)
    alpha = min(0.7, 0.999) * math.exp(-0.5 * d @ (conic @ d))
    pos = cam.position()
    rgb = O.eval_sh(sc.sh3[0], 0, -pos / np.linalg.norm(pos))
    for c in range(3):
        assert out[16, 16, c] == pytest.approx(rgb[c] * alpha + bg[c] * (1 - alpha), rel=1e-12)


def test_rasterize_matches_reference_render():
    """test_raster.cpp:157-168"""
    rng = O.Rng(43)
    for _ in range(10):
        scene = rng.random_scene(15, 15)
        cam = rng.random_camera()
        t = rng.uniform()
        a = O.rasterize(scene, cam, t, (0.2, 0.2, 0.2))["rgb"]
        b = O.reference_render(scene, cam, t, (0.2, 0.2, 0.2))
        assert np.abs(a - b).max() <= 1e-5


def test_bit_identical_across_threads():
    """test_raster.cpp:170-183"""
    rng = O.Rng(44)
    scene = rng.random_scene(40, 40)
    cam = rng.random_camera()
    a = O.rasterize(scene, cam, 0.37, (0, 0, 0), num_threads=1)["rgb"]
    b = O.rasterize(scene, cam, 0.37, (0, 0, 0), num_threads=4)["rgb"]
    c = O.rasterize(scene, cam, 0.37, (0, 0, 0), num_threads=8)["rgb"]
    assert (a == b).all() and (a == c).all()


def single_static_scene(opacity_logit=1.0):
    """One default Gaussian3D (scene.hpp:16-24) with the given opacity logit."""
    return HybridScene(mean3=np.zeros((1, 3)), quat3=np.array([[1.0, 0, 0, 0]]), log_s3=np.zeros((1, 3)),
                       op3=np.array([opacity_logit]))


def _boxes_expect(splats, w, h):
    expect = np.zeros((h, w), dtype=np.uint32)
    for sp in splats:
        expect[sp["y0"]:sp["y1"] + 1, sp["x0"]:sp["x1"] + 1] += 1
    return expect


def test_density_map_covers_exactly_the_boxes():
    """test_raster.cpp:185-201"""
    rng = O.Rng(45)
    scene = rng.random_scene(5, 5)
    cam = rng.random_camera(48, 48)
    counts = O.density_map(scene, cam, 0.5)
    assert counts.shape == (48, 48)
    assert (counts == _boxes_expect(O.project_scene(scene, cam, 0.5)[0], 48, 48)).all()
    dyn = O.density_map(scene, cam, 0.5, dynamics_only=True)
    assert (dyn <= counts).all()


def test_density_map_single_static():
    """tests/python/test_smoke.py:84-96"""
    scene = single_static_scene()
    cam = O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], 40.0, 24, 16)
    total = O.density_map(scene, cam, 0.5)
    dyn = O.density_map(scene, cam, 0.5, dynamics_only=True)
    assert total.shape == (16, 24)
    assert total.sum() > 0
    assert (dyn <= total).all() and dyn.sum() == 0


def test_range_and_finite():
    """test_raster.cpp:203-215"""
    rng = O.Rng(46)
    for _ in range(5):
        scene = rng.random_scene(20, 20)
        cam = rng.random_camera()
        out = O.rasterize(scene, cam, 0.5, (1.0, 1.0, 1.0))["rgb"]
        assert np.isfinite(out).all() and out.min() >= 0.0 and out.max() <= 1.0 + 1e-12


def test_acceptance_renderer_equivalence_sweep():
    """test_acceptance.cpp:111-141: random scenes <= 200 Gaussians at 64x64."""
    rng = O.Rng(7)
    for i in range(25):
        n = 10 + (i * 7) % 90
        scene = rng.random_scene(n, n)
        cam = rng.random_camera(64, 64)
        t = rng.uniform()
        a = O.rasterize(scene, cam, t, (0.2, 0.2, 0.2), num_threads=1)["rgb"]
        b = O.reference_render(scene, cam, t, (0.2, 0.2, 0.2))
        c = O.rasterize(scene, cam, t, (0.2, 0.2, 0.2), num_threads=4)["rgb"]
        assert np.abs(a - b).max() <= 1e-5
        assert (a == c).all()


def test_tiled_forward_train_equals_rasterize_and_untiled():
    """test_backward.cpp:98-100: forward_train == rasterize bitwise."""
    rng = O.Rng(45)
    for _ in range(4):
        scene = rng.random_scene(30, 30, 3)
        cam = rng.random_camera(48, 40)
        t = rng.uniform()
        ref = O.rasterize(scene, cam, t, (0.15, 0.2, 0.25))["rgb"]
        img, tape = O.forward_train(scene, cam, t, (0.15, 0.2, 0.25))
        img2, tape2 = O.forward_train(scene, cam, t, (0.15, 0.2, 0.25), untiled=True)
        assert (img == ref).all() and (img2 == ref).all()
        assert tape.contrib_total() == tape2.contrib_total()


def test_sorted_instances_order():
    """raster.cpp:180-212: instances sorted by (tile, f32 depth bits, prim index)."""
    rng = O.Rng(47)
    scene = rng.random_scene(50, 50)
    cam = rng.random_camera(96, 80)
    splats, _ = O.project_scene(scene, cam, 0.5)
    tiles, prims = O.sorted_instances(scene, cam, 0.5)
    key = tiles.astype(np.uint64) << np.uint64(32) | splats["depth_bits"][prims].astype(np.uint64)
    order = np.lexsort((prims, key))
    assert (order == np.arange(len(order))).all()
