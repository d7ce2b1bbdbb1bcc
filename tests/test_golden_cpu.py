"""Frozen fixtures (tests/golden/, written once by make_golden.py): the
product's host-side readers against a byte stream that no code under test
produced at run time."""
import hashlib
import json
import os

import numpy as np

from oracle import checkpoint as CK
from paper_2505_13215_b200 import api as A
from paper_2505_13215_b200 import dataset as D
from paper_2505_13215_b200.scene import HybridScene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELDS = HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS


def test_golden_checkpoint_integrity_and_decode():
    path = os.path.join(GOLDEN, "ckpt_small.hgsc")
    meta = json.load(open(os.path.join(GOLDEN, "ckpt_small.json")))
    raw = open(path, "rb").read()
    assert hashlib.sha256(raw).hexdigest() == meta["sha256"] and len(raw) == meta["bytes"]
    ref_scene, ref_state = CK.decode_checkpoint(raw)
    scene, state = A.load_checkpoint_full(path)
    assert (scene.n4, scene.n3, scene.sh_degree) == (meta["n4"], meta["n3"], meta["sh_degree"])
    assert (scene.tau, scene.duration_seconds, scene.extent) == (meta["tau"], meta["duration_seconds"], meta["extent"])
    assert (state.step, state.skipped_nonfinite) == (meta["step"], meta["skipped_nonfinite"])
    for f in FIELDS:
        assert np.array_equal(getattr(scene, f), getattr(ref_scene, f)), f
        assert np.array_equal(getattr(state.m, f), getattr(ref_state.m, f)), f
        assert np.array_equal(getattr(state.v, f), getattr(ref_state.v, f)), f
    assert np.array_equal(state.count4, ref_state.count4) and np.array_equal(state.grad_norm3, ref_state.grad_norm3)


def test_golden_checkpoint_rewrite(tmp_path):
    scene, state = A.load_checkpoint_full(os.path.join(GOLDEN, "ckpt_small.hgsc"))
    p = str(tmp_path / "again.hgsc")
    A.save_checkpoint(scene, p, state)
    ref_scene, ref_state = CK.decode_checkpoint(open(os.path.join(GOLDEN, "ckpt_small.hgsc"), "rb").read())
    assert open(p, "rb").read() == CK.encode_checkpoint(ref_scene, ref_state)


def test_golden_ppm():
    img = D.read_ppm_u8(os.path.join(GOLDEN, "frame_5x3.ppm"))
    assert img.shape == (3, 5, 3)
    assert img.tobytes() == bytes([(7 * i + 3) % 256 for i in range(45)])
