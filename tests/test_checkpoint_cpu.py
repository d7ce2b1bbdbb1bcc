"""Host-scene checkpoints through the C ABI (no GPU): byte-identical to the
format restatement (oracle/checkpoint.py, data_io.cpp:444-719) and the
reference's error taxonomy (test_data_io.cpp:119-160)."""
import numpy as np
import pytest

import oracle as O
from oracle import checkpoint as CK
from paper_2505_13215_b200 import api as A
from paper_2505_13215_b200.scene import HybridScene

from .test_oracle_checkpoint import canonical, random_state, scenes_identical


def to_api_state(st):
    return A.CheckpointState(m=st.m, v=st.v, grad_norm4=st.grad_norm4, grad_norm3=st.grad_norm3, count4=st.count4,
                             count3=st.count3, step=st.step, skipped_nonfinite=st.skipped_nonfinite)


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_host_write_matches_format(tmp_path, deg):
    scene = O.Rng(200 + deg).random_scene(23, 17, deg)
    scene.tau, scene.duration_seconds, scene.extent = 0.37, 2.5, 3.1
    st = random_state(scene, deg)
    p = tmp_path / "a.hgsc"
    A.save_checkpoint(scene, str(p), to_api_state(st))
    assert p.read_bytes() == CK.encode_checkpoint(scene, st)
    A.save_checkpoint(scene, str(p))
    assert p.read_bytes() == CK.encode_checkpoint(scene)


def test_host_read_roundtrip(tmp_path):
    """test_data_io.cpp:85-117 through the product's host reader"""
    scene = O.Rng(101).random_scene(50, 50, 2)
    scene.tau, scene.duration_seconds, scene.extent = 0.37, 2.5, 3.1
    st = random_state(scene)
    p = str(tmp_path / "a.hgsc")
    CK.save_checkpoint(scene, st, p)
    back, bst = A.load_checkpoint_full(p)
    assert scenes_identical(canonical(scene), back)
    assert bst.step == 1234 and bst.skipped_nonfinite == 7
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        assert np.array_equal(getattr(bst.m, f), getattr(st.m, f)) and np.array_equal(getattr(bst.v, f), getattr(st.v, f))
    assert np.array_equal(bst.grad_norm3, st.grad_norm3) and np.array_equal(bst.grad_norm4, st.grad_norm4)
    assert np.array_equal(bst.count3, st.count3) and np.array_equal(bst.count4, st.count4)
    p2 = str(tmp_path / "b.hgsc")
    A.save_checkpoint(scene, p2)
    assert A.load_checkpoint_full(p2)[1] is None
    assert scenes_identical(canonical(scene), A.load_checkpoint(p2))


def test_host_errors(tmp_path):
    scene = O.Rng(102).random_scene(8, 8)
    good = CK.encode_checkpoint(scene)
    p = tmp_path / "x.hgsc"

    def load(b):
        p.write_bytes(bytes(b))
        return A.load_checkpoint(str(p))

    bad = bytearray(good)
    bad[len(bad) // 2] ^= 1
    with pytest.raises(A.IntegrityError):
        load(bad)
    for keep in (len(good) - 1, len(good) // 2, 10, 6, 2):
        with pytest.raises(A.FormatError):
            load(good[:keep])
    bad = bytearray(good)
    bad[0] = ord("X")
    with pytest.raises(A.FormatError):
        load(bad)
    bad = bytearray(good)
    bad[4] = 99
    with pytest.raises(A.UnsupportedVersionError):
        load(bad)
    with pytest.raises(A.FormatError):
        A.load_checkpoint(str(tmp_path / "nope.hgsc"))
    s2 = scene.copy()
    s2.ql[1] = [0.0, 0.0, 0.0, 3.0]
    with pytest.raises(A.FormatError, match="non-unit"):
        load(CK.encode_checkpoint(s2))
    st = random_state(scene)
    st.count4 = st.count4[:-2]
    with pytest.raises(A.FormatError, match="disagrees"):
        load(CK.encode_checkpoint(scene, st))


def test_empty_scene(tmp_path):
    scene = HybridScene(sh_degree=1, tau=0.2, duration_seconds=4.0, extent=2.0)
    p = str(tmp_path / "e.hgsc")
    A.save_checkpoint(scene, p, A.CheckpointState.zeros_like(scene))
    assert open(p, "rb").read() == CK.encode_checkpoint(scene, CK.State(scene))
    back, st = A.load_checkpoint_full(p)
    assert back.n3 == 0 and back.n4 == 0 and back.duration_seconds == 4.0 and st is not None
