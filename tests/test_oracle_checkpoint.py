"""Pins the checkpoint restatement (oracle/checkpoint.py) against the
reference's test_data_io.cpp:85-160 cases and the hand-assembled layout."""
import struct
import zlib

import numpy as np
import pytest

import oracle as O
from oracle import checkpoint as CK
from paper_2505_13215_b200.scene import HybridScene, sh_coeff_count


def random_state(scene, seed=0):
    """test_data_io.cpp:59-81 (values from numpy, same shapes)."""
    rng = np.random.default_rng(seed)
    st = CK.State(scene)
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        getattr(st.m, f)[...] = rng.uniform(-1, 1, getattr(scene, f).shape)
        getattr(st.v, f)[...] = np.abs(rng.uniform(-1, 1, getattr(scene, f).shape))
    st.grad_norm3 = np.abs(rng.uniform(-1, 1, scene.n3))
    st.grad_norm4 = np.abs(rng.uniform(-1, 1, scene.n4))
    st.count3 = rng.integers(0, 100, scene.n3).astype(np.uint32)
    st.count4 = rng.integers(0, 100, scene.n4).astype(np.uint32)
    st.step, st.skipped_nonfinite = 1234, 7
    return st


def scenes_identical(a, b):
    if (a.n3, a.n4, a.sh_degree, a.tau, a.duration_seconds, a.extent) != \
            (b.n3, b.n4, b.sh_degree, b.tau, b.duration_seconds, b.extent):
        return False
    return all(np.array_equal(getattr(a, f), getattr(b, f)) for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS)


def canonical(scene):
    """the loader flips quaternions to the w >= 0 hemisphere (data_io.cpp:506-508)"""
    s = scene.copy()
    for f in ("quat3", "ql", "qr"):
        q = getattr(s, f)
        for i in range(q.shape[0]):
            w, x, y, z = q[i]
            if w < 0 or (w == 0 and (x < 0 or (x == 0 and (y < 0 or (y == 0 and z < 0))))):
                q[i] = -q[i]
    return s


def test_roundtrip_bit_exact_with_state(tmp_path):
    """test_data_io.cpp:85-117"""
    scene = O.Rng(101).random_scene(50, 50, 2)
    scene.tau, scene.duration_seconds, scene.extent = 0.37, 2.5, 3.1
    st = random_state(scene)
    p = str(tmp_path / "a.hgsc")
    CK.save_checkpoint(scene, st, p)
    back, bst = CK.load_checkpoint(p)
    assert scenes_identical(canonical(scene), back)
    assert bst.step == 1234 and bst.skipped_nonfinite == 7
    assert np.array_equal(bst.m.mean3, st.m.mean3) and np.array_equal(bst.v.sh4, st.v.sh4)
    assert np.array_equal(bst.grad_norm4, st.grad_norm4) and np.array_equal(bst.count3, st.count3)
    p2, p3 = str(tmp_path / "b.hgsc"), str(tmp_path / "c.hgsc")
    CK.save_checkpoint(scene, None, p2)
    bare, none = CK.load_checkpoint(p2)
    assert none is None and scenes_identical(canonical(scene), bare)
    CK.save_checkpoint(scene, None, p3)
    assert open(p2, "rb").read() == open(p3, "rb").read()


def test_layout_by_hand():
    """One static + one dynamic, degree 0: every byte where data_io.cpp puts it."""
    s = HybridScene(sh_degree=0, tau=0.5, duration_seconds=2.0, extent=1.5,
                    mean_x=[[1.0, 2.0, 3.0]], mean_t=[0.25], ql=[[1.0, 0, 0, 0]], qr=[[0, 1.0, 0, 0]],
                    log_s4=[[-1.0, -2.0, -3.0, -4.0]], op4=[0.5], sh4=[[[0.1, 0.2, 0.3]]],
                    mean3=[[4.0, 5.0, 6.0]], quat3=[[0, 0, 1.0, 0]], log_s3=[[-5.0, -6.0, -7.0]], op3=[0.75],
                    sh3=[[[0.4, 0.5, 0.6]]])
    b = CK.encode_checkpoint(s)
    payload = struct.pack("<Idddqq", 0, 0.5, 2.0, 1.5, 1, 1)
    payload += struct.pack("<11d", 4, 5, 6, 0, 0, 1, 0, -5, -6, -7, 0.75) + struct.pack("<I", 0) + \
        struct.pack("<3d", 0.4, 0.5, 0.6)
    payload += struct.pack("<17d", 1, 2, 3, 0.25, 1, 0, 0, 0, 0, 1, 0, 0, -1, -2, -3, -4, 0.5) + \
        struct.pack("<I", 0) + struct.pack("<3d", 0.1, 0.2, 0.3)
    assert b == b"HGSC" + struct.pack("<I", 1) + b"SCEN" + struct.pack("<QI", len(payload), zlib.crc32(payload)) + \
        payload
    assert len(payload) == 44 + (92 + 24) + (140 + 24)


def test_corruption_and_truncation(tmp_path):
    """test_data_io.cpp:119-160"""
    scene = O.Rng(102).random_scene(8, 8)
    good = CK.encode_checkpoint(scene)
    assert len(good) > 64
    bad = bytearray(good)
    bad[len(bad) // 2] ^= 0x01
    with pytest.raises(CK.IntegrityError):
        CK.decode_checkpoint(bytes(bad))
    for keep in (len(good) - 1, len(good) // 2, 10):
        with pytest.raises(CK.FormatError):
            CK.decode_checkpoint(good[:keep])
    bad = bytearray(good)
    bad[0] = ord("X")
    with pytest.raises(CK.FormatError):
        CK.decode_checkpoint(bytes(bad))
    bad = bytearray(good)
    bad[4] = 99
    with pytest.raises(CK.UnsupportedVersionError):
        CK.decode_checkpoint(bytes(bad))
    with pytest.raises(CK.FormatError):
        CK.load_checkpoint(str(tmp_path / "nope.hgsc"))


def test_unknown_section_skipped_and_nonunit_quat():
    scene = O.Rng(103).random_scene(4, 4)
    good = CK.encode_checkpoint(scene)
    extra = b"XTRA" + struct.pack("<QI", 3, zlib.crc32(b"abc")) + b"abc"
    back, _ = CK.decode_checkpoint(good + extra)
    assert scenes_identical(canonical(scene), back)
    s2 = scene.copy()
    s2.quat3[0] = [2.0, 0, 0, 0]
    with pytest.raises(CK.FormatError):
        CK.decode_checkpoint(CK.encode_checkpoint(s2))


def test_state_must_match_scene():
    scene = O.Rng(104).random_scene(6, 5, 1)
    st = random_state(scene)
    st.grad_norm4 = st.grad_norm4[:-1]
    with pytest.raises(CK.FormatError):
        CK.decode_checkpoint(CK.encode_checkpoint(scene, st))
    assert sh_coeff_count(1) == 4
