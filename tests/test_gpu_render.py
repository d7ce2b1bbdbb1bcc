"""GPU render parity: the sm_100a path against the FP64 oracle, through the C ABI.

Gates (BASELINE.json north_star / SURVEY.md 8d):
  * bit-exact: projected set, f32 depth bits, pixel boxes (hence tile
    assignment), the full tile-sorted instance order, RenderStats;
  * image: max |delta| <= 1e-4 and PSNR > 60 dB against the oracle.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200.scene import HybridScene, ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4  # max abs error vs the FP64 oracle (north_star)
PSNR_MIN = 60.0


@pytest.fixture(scope="module")
def ctx():
    from paper_2505_13215_b200.api import Context

    c = Context(0)
    c.debug_keep_instances(True)  # keep the reference's full instance list for the parity check
    yield c
    c.close()


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b) ** 2))
    return math.inf if mse == 0 else 10 * math.log10(1.0 / mse)


def check_render(ctx, scene, cam, t, bg=(0.2, 0.2, 0.2), cutoff=0.05, threads=8):
    scene = scene.as_float32_exact()
    ctx.upload(scene)
    out = ctx.render(cam, t, bg, weight_cutoff=cutoff, count_map=True, transmittance_map=True)
    ref = O.rasterize(scene, cam, t, bg, num_threads=threads, weight_cutoff=cutoff, count_map=True,
                      transmittance_map=True)
    assert out["stats"] == ref["stats"]
    # bit-exact projection: set, depth key, box
    sp = ctx.debug_splats()
    rs, _ = O.project_scene(scene, cam, t, cutoff)
    assert (sp["gid"] == rs["gid"]).all()
    assert (sp["depth_bits"] == rs["depth_bits"]).all()
    assert (sp["box"] == np.stack([rs["x0"], rs["x1"], rs["y0"], rs["y1"]], 1)).all()
    # bit-exact tile-sorted instance order
    tiles, gids = ctx.debug_instances()
    rt, rp = O.sorted_instances(scene, cam, t, cutoff)
    assert len(tiles) == len(rt)
    assert (tiles == rt).all()
    assert (gids == rs["gid"][rp]).all()
    # conic / alpha within FP64 rounding of the oracle
    assert np.abs(sp["mean"] - np.stack([rs["sx"], rs["sy"]], 1)).max(initial=0) < 1e-9
    assert np.abs(sp["alpha"] - rs["alpha"]).max(initial=0) < 1e-12
    # image
    err = np.abs(out["rgb"].astype(np.float64) - ref["rgb"]).max()
    assert err <= IMG_TOL, err
    assert psnr(out["rgb"], ref["rgb"]) > PSNR_MIN
    assert (out["counts"] == ref["counts"]).all()
    assert np.abs(out["transmittance"] - ref["transmittance"]).max() <= 1e-4
    return out, ref


def test_empty_scene_is_background(ctx):
    cam = O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], 50.0, 32, 32)
    ctx.upload(HybridScene())
    out = ctx.render(cam, 0.3, (0.1, 0.5, 0.9))
    assert np.allclose(out["rgb"], np.array([0.1, 0.5, 0.9], dtype=np.float32))


@pytest.mark.parametrize("seed", [43, 44, 45, 46])
def test_random_mixed_scenes_match_oracle(ctx, seed):
    rng = O.Rng(seed)
    for _ in range(3):
        scene = rng.random_scene(15, 15)
        cam = rng.random_camera()
        check_render(ctx, scene, cam, rng.uniform())


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_sh_degrees(ctx, deg):
    rng = O.Rng(100 + deg)
    scene = rng.random_scene(60, 60, deg)
    cam = rng.random_camera(96, 72)
    check_render(ctx, scene, cam, 0.5)


def test_statics_only_and_dynamics_only(ctx):
    rng = O.Rng(7)
    check_render(ctx, rng.random_scene(80, 0, 1), rng.random_camera(80, 64), 0.2)
    check_render(ctx, rng.random_scene(0, 80, 1), rng.random_camera(80, 64), 0.9)


def test_edge_sizes_and_tile_boundaries(ctx):
    """Images that are not a multiple of the 16-px tile, 1-px images."""
    rng = O.Rng(8)
    scene = rng.random_scene(40, 40, 2)
    for w, h in [(1, 1), (17, 33), (33, 17), (129, 5)]:
        cam = rng.random_camera(w, h)
        check_render(ctx, scene, cam, 0.4)


def test_culling_paths(ctx):
    """Depth, temporal and degenerate-temporal culls counted like the reference."""
    rng = O.Rng(9)
    scene = rng.random_scene(20, 40, 1)
    scene.log_s4[:5, :] = math.log(1e-7)  # Sigma_tt ~ 1e-14 -> degenerate_temporal
    scene.mean_x[5:8] = [[0.0, 0.0, -40.0]] * 3  # behind / far
    cam = rng.random_camera(64, 64)
    out, ref = check_render(ctx, scene, cam, 0.5)
    assert ref["stats"]["degenerate_temporal"] >= 1


def test_invalid_camera_raises(ctx):
    from paper_2505_13215_b200.api import Context  # noqa: F401

    cam = O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], 50.0, 32, 32)
    cam.fx = -1.0
    ctx.upload(HybridScene())
    with pytest.raises(ValueError):
        ctx.render(cam, 0.0)


def test_dense_scene_many_instances(ctx):
    """Crowded tiles (hundreds of splats per tile, early termination, fix-ups)."""
    scene = synthetic_scene(3000, 1000, 3, seed=11, density_n=100)
    cam = ring_camera(11, 160, 120)
    check_render(ctx, scene, cam, 0.5)


def test_c1_config_parity(ctx):
    """configs[0]: 100k 4D Gaussians, 640x480, t = 0.5 (BASELINE.json)."""
    scene = synthetic_scene(100_000, 0, 3, seed=1)
    cam = ring_camera(1, 640, 480)
    out, ref = check_render(ctx, scene, cam, 0.5)
    info = ctx.render_info()
    assert info["instances"] > 0


def test_drop_in_rasterize_float64(ctx):
    """hgs_rasterize: host double scene in, host double image out."""
    from paper_2505_13215_b200.api import rasterize

    rng = O.Rng(12)
    scene = rng.random_scene(30, 30, 1).as_float32_exact()
    cam = rng.random_camera(64, 48)
    img = rasterize(scene, cam, 0.3, (0.1, 0.2, 0.3))
    ref = O.rasterize(scene, cam, 0.3, (0.1, 0.2, 0.3))["rgb"]
    assert img.dtype == np.float64 and img.shape == (48, 64, 3)
    assert np.abs(img - ref).max() <= IMG_TOL


def test_render_deterministic(ctx):
    scene = synthetic_scene(20000, 5000, 3, seed=3)
    cam = ring_camera(3, 320, 240)
    ctx.upload(scene)
    a = ctx.render(cam, 0.5)["rgb"]
    b = ctx.render(cam, 0.5)["rgb"]
    assert (a == b).all()


def test_cpp_consumer_runs(tmp_path):
    """examples/render_demo.cpp through the C ABI: the single-splat closed form."""
    import subprocess

    from tests.test_capi_cpu import _build_demo

    out = subprocess.run([_build_demo(tmp_path)], capture_output=True, text=True, check=True).stdout
    assert "projected=1" in out
    vals = [float(v) for v in out.split("centre=(")[1].rstrip(")\n").split(",")]
    cov = O.build_cov3(np.eye(3), [math.log(0.3)] * 3)
    cam = O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], 40.0, 33, 33)
    s = O.project_3d([0, 0, 0], cov, cam)
    d = np.array([16.5, 16.5]) - np.array([s["sx"], s["sy"]])
    alpha = 0.7 * math.exp(-0.5 * d @ (np.array(s["conic"]).reshape(2, 2) @ d))
    for c, (rgb, bgc) in enumerate(zip((0.9, 0.1, 0.3), (0.0, 0.0, 1.0))):
        assert vals[c] == pytest.approx(rgb * alpha + bgc * (1 - alpha), abs=1e-6)


def test_c2_config_parity(ctx):
    """configs[1] at full size: 240k 4D + 60k 3D Gaussians, SH 3, 1352x1014 --
    every projected splat, the complete tile-sorted instance list (~3.8M) and
    the image against the oracle."""
    scene = synthetic_scene(240_000, 60_000, 3, seed=2, tau=0.5)
    cam = ring_camera(2, 1352, 1014, index=5, n_ring=16)
    check_render(ctx, scene, cam, 1.0 / 3.0, threads=O.hardware_threads())
    info = ctx.render_info()
    assert info["instances"] > 1_000_000 and info["kept_instances"] < info["instances"]


@pytest.mark.parametrize("cfg", ["dense", "c2"])
def test_fused_duplication_path_matches_debug_path(ctx, cfg):
    """The production path (duplication + exact culling + compaction fused,
    look-back ordered) renders bit-identically to the path that keeps the
    reference's full instance list (used by the other parity tests)."""
    from paper_2505_13215_b200.api import Context

    if cfg == "dense":
        scene, cam = synthetic_scene(3000, 1000, 3, seed=11, density_n=100), ring_camera(11, 160, 120)
    else:
        scene, cam = synthetic_scene(240_000, 60_000, 3, seed=2), ring_camera(2, 1352, 1014, index=3, n_ring=16)
    prod = Context(0)
    try:
        ctx.upload(scene)
        prod.upload(scene)
        a = ctx.render(cam, 0.4, (0.2, 0.2, 0.2), transmittance_map=True)
        b = prod.render(cam, 0.4, (0.2, 0.2, 0.2), transmittance_map=True)
        assert (a["rgb"] == b["rgb"]).all() and (a["transmittance"] == b["transmittance"]).all()
        assert ctx.render_info() == prod.render_info()
    finally:
        prod.close()


@pytest.mark.parametrize("seed,size,t", [(3, (320, 240), 0.45), (5, (256, 192), 0.8), (7, (200, 150), 0.1)])
def test_quadrant_masks_are_conservative(ctx, seed, size, t):
    """The 8x8-quadrant masks (band test / exact rectangle test of the
    duplication kernels) never clear a quadrant in which some pixel of the
    splat's box reaches alpha >= 1/255 (raster.cpp:139-140, FP64 truth)."""
    from paper_2505_13215_b200.scene import synthetic_scene as syn

    scene = syn(15000, 5000, sh_degree=1, seed=seed).as_float32_exact()
    cam = ring_camera(seed, *size)
    ctx.upload(scene)
    ctx.debug_keep_instances(True)  # (the module's context keeps the full list anyway)
    ctx.render(cam, t)
    tiles, gids = ctx.debug_instances()
    masks = ctx.debug_instance_masks()
    sp = ctx.debug_splats()
    pos = np.full(int(sp["gid"].max()) + 1, -1, np.int64)
    pos[sp["gid"]] = np.arange(len(sp["gid"]))
    k = pos[gids]
    tiles_x = (cam.width + 15) // 16
    tx, ty = tiles.astype(np.int64) % tiles_x, tiles.astype(np.int64) // tiles_x
    box = sp["box"][k]  # x0, x1, y0, y1
    mx, my = sp["mean"][k, 0], sp["mean"][k, 1]
    c = sp["conic"][k]
    lnc = np.log(sp["alpha"][k] * 255.0)  # reachable iff power <= ln(255 alpha)
    off = np.arange(8)
    bad = 0
    for q in range(4):
        qx0 = tx * 16 + (q & 1) * 8
        qy0 = ty * 16 + (q >> 1) * 8
        px = qx0[:, None] + off[None, :]  # (n, 8)
        py = qy0[:, None] + off[None, :]
        inx = (px >= box[:, 0:1]) & (px <= box[:, 1:2]) & (px < cam.width)
        iny = (py >= box[:, 2:3]) & (py <= box[:, 3:4]) & (py < cam.height)
        dx = (px + 0.5) - mx[:, None]
        dy = (py + 0.5) - my[:, None]
        pw = 0.5 * (c[:, 0, None, None] * dx[:, None, :] ** 2 + (c[:, 1] + c[:, 2])[:, None, None] * dx[:, None, :] *
                    dy[:, :, None] + c[:, 3, None, None] * dy[:, :, None] ** 2)  # (n, y, x)
        ok = inx[:, None, :] & iny[:, :, None] & (pw <= lnc[:, None, None])
        reach = ok.any(axis=(1, 2))
        bad += int((reach & ((masks >> q) & 1 == 0)).sum())
    assert bad == 0, bad
    assert masks.any()


def _replicate3(scene, idx):
    from dataclasses import replace

    return replace(scene, mean3=scene.mean3[idx], quat3=scene.quat3[idx], log_s3=scene.log_s3[idx],
                   op3=scene.op3[idx], sh3=scene.sh3[idx])


def test_depth_sort_ties_and_clusters(ctx):
    """Depth-sort corner cases: 6000 copies of 3 Gaussians (equal depth keys:
    ties broken by the projected index), a narrow depth cluster in front of
    one far outlier (keys sharing their high digits) and a spread scene --
    all against the oracle's instance order."""
    rng = O.Rng(12)
    base = rng.random_scene(3, 0, 1)
    cam = rng.random_camera(48, 40)
    check_render(ctx, _replicate3(base, np.arange(6000) % 3), cam, 0.5)
    cl = rng.random_scene(3000, 0, 0)
    cl.mean3[:] = 1e-3 * (cl.mean3 - cl.mean3.mean(0))
    cl.mean3[0] = [0.0, 0.0, 5.0]  # 8 units away, the cluster at 3
    check_render(ctx, cl, O.look_at([0, 0, -3], [0, 0, 0], [0, -1, 0], 50.0, 48, 40), 0.5)
    check_render(ctx, synthetic_scene(20_000, 20_000, 0, seed=13), ring_camera(13, 96, 80), 0.5)
