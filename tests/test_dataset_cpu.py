"""Dataset ingest on the host: PPM frames through the C ABI
(image.cpp:35-75), the multi-view directory format (data_io.cpp:44-187) and
the reference's test_data_io.cpp cases for them; init_scene's oracle
(data_io.cpp:189-238, test_data_io.cpp:232-275)."""
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200 import dataset as D
from paper_2505_13215_b200.scene import Camera, ring_camera
from paper_2505_13215_b200.train import SRGB8_LUT, Frame, MultiViewDataset, linear_to_srgb8, quantize_8bit


def test_ppm_roundtrip_pixel_exact_after_quantization(tmp_path):
    """test_data_io.cpp:162-177"""
    rng = np.random.default_rng(103)
    img = rng.uniform(0, 1, (9, 17, 3))
    p = str(tmp_path / "img.ppm")
    D.write_ppm(img, p)
    back = D.read_ppm(p)
    assert back.shape == (9, 17, 3)
    assert np.array_equal(back, quantize_8bit(img))
    assert np.array_equal(quantize_8bit(quantize_8bit(img)), quantize_8bit(img))
    assert np.array_equal(D.read_ppm_u8(p), linear_to_srgb8(img))
    D.write_ppm(img.astype(np.float32), p)  # float frames quantise the same way
    assert np.array_equal(D.read_ppm_u8(p), linear_to_srgb8(img.astype(np.float32).astype(np.float64)))
    D.write_ppm(D.read_ppm_u8(p), str(tmp_path / "u8.ppm"))  # u8 codes are written as they are
    assert open(p, "rb").read() == open(str(tmp_path / "u8.ppm"), "rb").read()


def test_ppm_header_rules(tmp_path):
    pix = bytes(range(2 * 3 * 3))
    ok = [b"P6\n3 2\n255\n", b"P6 3 2 255 ", b"P6\n# comment\n3 # w\n#\n2\n255\n", b"  P6\t3\n2\r255\n"]
    for i, hdr in enumerate(ok):
        p = tmp_path / f"ok{i}.ppm"
        p.write_bytes(hdr + pix + b"trailing bytes are ignored")
        assert D.ppm_info(str(p)) == (3, 2)
        assert D.read_ppm_u8(str(p)).tobytes() == pix
    long_comment = b"P6\n#" + b"x" * 200000 + b"\n3 2\n255\n"
    p = tmp_path / "long.ppm"
    p.write_bytes(long_comment + pix)
    assert D.read_ppm_u8(str(p)).tobytes() == pix
    bad = {"magic.ppm": b"P5\n3 2\n255\n" + pix, "maxval.ppm": b"P6\n3 2\n65535\n" + pix,
           "zero.ppm": b"P6\n0 2\n255\n", "neg.ppm": b"P6\n3 -2\n255\n", "nodigits.ppm": b"P6\nx 2\n255\n",
           "trunc.ppm": b"P6\n3 2\n255\n" + pix[:-1], "nobyte.ppm": b"P6\n3 2\n255", "empty.ppm": b""}
    for name, content in bad.items():
        p = tmp_path / name
        p.write_bytes(content)
        with pytest.raises(D.FormatError):
            D.read_ppm_u8(str(p))
    with pytest.raises(D.FormatError, match="cannot open"):
        D.read_ppm_u8(str(tmp_path / "missing.ppm"))


def test_ppm_batch_parallel(tmp_path):
    rng = np.random.default_rng(7)
    imgs = rng.integers(0, 256, (24, 13, 11, 3), dtype=np.uint8)
    paths = []
    for i, im in enumerate(imgs):
        paths.append(str(tmp_path / f"f{i}.ppm"))
        D.write_ppm(im, paths[-1])
    out = D.read_ppm_batch(paths, 11, 13, threads=4)
    assert np.array_equal(out, imgs)
    assert np.array_equal(D.read_ppm_batch(paths, 11, 13, threads=1), imgs)
    open(paths[5], "wb").write(b"P6\n11 13\n255\n")  # truncated
    open(paths[9], "wb").write(b"P5\n")
    with pytest.raises(D.FormatError, match="f5.ppm"):  # the first failing frame, in order
        D.read_ppm_batch(paths, 11, 13, threads=8)
    with pytest.raises(D.FormatError, match="differs"):
        D.read_ppm_batch(paths[:2], 12, 13)


def test_key_value_file(tmp_path):
    p = tmp_path / "meta.txt"
    p.write_text("# header\nduration_seconds = 2.5  # trailing\n\nbackground_r=0.25\n")
    kv = D.KeyValueFile(str(p))
    assert kv.get_float("duration_seconds", 1.0) == 2.5
    assert kv.get_float("background_g", 0.5) == 0.5
    with pytest.raises(D.FormatError, match="unknown keys: background_r"):
        kv.finish()
    for content, msg in (("a\n", "expected key=value"), ("a =\n", "empty key"), ("a=1\na=2\n", "duplicate key")):
        p.write_text(content)
        with pytest.raises(D.FormatError, match=msg):
            D.KeyValueFile(str(p))
    p.write_text("n = x\n")
    with pytest.raises(D.FormatError, match="not a number"):
        D.KeyValueFile(str(p)).get_float("n", 0.0)


def test_points_roundtrip(tmp_path):
    """test_data_io.cpp:232-250"""
    rng = np.random.default_rng(105)
    pts = D.InitPoints(rng.uniform(-2, 2, (30, 3)), rng.uniform(0, 1, (30, 3)))
    p = str(tmp_path / "points.txt")
    D.save_points(pts, p)
    back = D.load_points(p)
    assert len(back) == 30
    assert np.array_equal(back.positions, pts.positions) and np.array_equal(back.rgb, pts.rgb)  # %.17g is exact
    with open(p, "a") as f:
        f.write("1 2 3\n")
    with pytest.raises(D.FormatError, match="expected x y z r g b"):
        D.load_points(p)


def small_dataset(n_cams=3, n_frames=3, w=24, h=20, seed=11):
    rng = np.random.default_rng(seed)
    cams = [ring_camera(i, w, h) for i in range(n_cams)]
    frames = [[Frame(time=j / (n_frames - 1), image=quantize_8bit(rng.uniform(0, 1, (h, w, 3))))
               for j in range(n_frames)] for _ in cams]
    pts = D.InitPoints(rng.uniform(-1, 1, (20, 3)), rng.uniform(0, 1, (20, 3)))
    return MultiViewDataset(cameras=cams, frames=frames, background=(0.1, 0.2, 0.3), duration_seconds=2.0,
                            camera_ids=list(range(n_cams)), init_points=pts)


def test_dataset_roundtrip(tmp_path):
    """test_data_io.cpp:192-230"""
    ds = small_dataset()
    root = str(tmp_path / "ds")
    D.save_dataset(ds, root)
    train, held = D.load_dataset(root, held_out_camera=2, frames="linear")
    assert len(train.cameras) == 2 and len(held.cameras) == 1 and held.camera_ids == [2]
    assert train.duration_seconds == 2.0 and train.background == (0.1, 0.2, 0.3)
    assert len(train.init_points) == 20 and np.array_equal(train.init_points.positions, ds.init_points.positions)
    for c, cid in enumerate(train.camera_ids):
        a, b = train.cameras[c], ds.cameras[cid]
        assert np.abs(a.rot - b.rot).max() < 1e-12 and np.abs(a.trans - b.trans).max() < 1e-12
        assert (a.fx, a.fy, a.cx, a.cy, a.width, a.height, a.near, a.far) == \
            (b.fx, b.fy, b.cx, b.cy, b.width, b.height, b.near, b.far)
        for f, fr in enumerate(train.frames[c]):
            assert fr.time == pytest.approx(ds.frames[cid][f].time)
            assert np.array_equal(fr.image, ds.frames[cid][f].image)  # quantised before saving: exact
    t8, _ = D.load_dataset(root, frames="u8", pinned=False, threads=2)
    assert t8.frames[0][0].image.dtype == np.uint8
    assert np.array_equal(SRGB8_LUT[t8.frames[1][2].image], ds.frames[1][2].image)
    with pytest.raises(D.FormatError, match="held-out camera id 99"):
        D.load_dataset(root, 99)
    with pytest.raises(D.FormatError):
        D.load_dataset(str(tmp_path / "missing"), -1)


def test_dataset_format_errors(tmp_path):
    ds = small_dataset(n_cams=2, n_frames=2)
    root = tmp_path / "ds"
    D.save_dataset(ds, str(root))
    with pytest.raises(D.FormatError, match="holding out the only camera"):
        one = tmp_path / "one"
        D.save_dataset(small_dataset(n_cams=1, n_frames=2), str(one))
        D.load_dataset(str(one), 0)
    os.remove(root / "cam01" / "frame_00001.ppm")
    with pytest.raises(D.FormatError, match="frame count differs"):
        D.load_dataset(str(root))
    D.save_dataset(ds, str(root))
    D.write_ppm(np.zeros((5, 5, 3)), str(root / "cam00" / "frame_00000.ppm"))
    with pytest.raises(D.FormatError, match="frame size disagrees"):
        D.load_dataset(str(root))
    D.save_dataset(ds, str(root))
    txt = (root / "cameras.txt").read_text().splitlines()
    (root / "cameras.txt").write_text("# comment line\n" + txt[0] + "\n" + " ".join(txt[1].split()[:10]) + "\n")
    with pytest.raises(D.FormatError, match="cameras.txt:3: expected"):
        D.load_dataset(str(root))
    bad = txt[1].split()
    bad[1] = "-5"
    (root / "cameras.txt").write_text(txt[0] + "\n" + " ".join(bad) + "\n")
    with pytest.raises(D.FormatError, match="fx, fy must be positive"):
        D.load_dataset(str(root))
    (root / "cameras.txt").write_text(txt[0] + "\n")
    (root / "meta.txt").write_text("duration_seconds = 1\ncolour = 3\n")
    with pytest.raises(D.FormatError, match="unknown keys: colour"):
        D.load_dataset(str(root))


def test_oracle_init_scene_shape():
    """test_data_io.cpp:252-275 on the oracle"""
    rng = np.random.default_rng(105)
    pos, rgb = rng.uniform(-2, 2, (30, 3)), rng.uniform(0, 1, (30, 3))
    s = O.init_scene(pos, rgb, sh_degree=1, tau=0.4, duration_seconds=3.0)
    assert s.n3 == 0 and s.n4 == 30 and s.tau == 0.4 and s.duration_seconds == 3.0 and s.sh_degree == 1
    assert s.extent > 0.0
    assert np.array_equal(s.mean_x, pos)
    assert np.allclose(np.exp(s.log_s4[:, 3]), 0.1)
    assert all(not O.is_static(ls, 0.4) for ls in s.log_s4[:, 3])
    assert np.allclose(1 / (1 + np.exp(-s.op4)), 0.1)
    assert (s.mean_t >= 0).all() and (s.mean_t <= 1).all()
    # 3-NN mean distance, brute force in numpy
    d = np.sqrt(((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(d, np.inf)
    nn = np.sort(d, axis=1)[:, :3].mean(1)
    assert np.allclose(s.log_s4[:, 0], np.log(np.maximum(nn, 1e-4)), rtol=1e-12)
    assert np.allclose(s.sh4[:, 0, :], (rgb - 0.5) / 0.28209479177387814)
    with pytest.raises(ValueError):
        O.init_scene(pos[:3], rgb[:3])
    assert math.isfinite(s.extent)


def test_camera_struct_roundtrip_via_text(tmp_path):
    cam = Camera.look_at([0.3, -1, -4], [0, 0, 0], [0, -1, 0], 71.5, 33, 21)
    ds = MultiViewDataset(cameras=[cam], frames=[[Frame(0.0, np.zeros((21, 33, 3)))]], camera_ids=[7])
    D.save_dataset(ds, str(tmp_path / "c"))
    t, _ = D.load_dataset(str(tmp_path / "c"))
    assert t.camera_ids == [7]
    assert np.array_equal(t.cameras[0].rot, cam.rot) and np.array_equal(t.cameras[0].trans, cam.trans)  # %.17g
