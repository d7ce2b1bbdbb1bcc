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


# ---- the oracle against outputs of the REFERENCE itself (tests/golden/
# make_ref_golden.py: the reference's own sources compiled here, oracle/_ref)
import oracle as O  # noqa: E402
import sys as _sys  # noqa: E402

_sys.path.insert(0, GOLDEN)
import make_ref_golden as RG  # noqa: E402

_REF = np.load(os.path.join(GOLDEN, "ref_golden.npz"))


def test_oracle_render_equals_reference_outputs():
    scene, cam = RG.case_render()
    a = O.rasterize(scene, cam, 0.4, RG.BG, count_map=True, transmittance_map=True)
    assert np.array_equal(a["rgb"], _REF["render_rgb"])
    assert np.array_equal(a["counts"], _REF["render_counts"])
    assert np.array_equal(a["transmittance"], _REF["render_trans"])
    assert [a["stats"][k] for k in sorted(a["stats"])] == list(_REF["render_stats"])
    sp, _ = O.project_scene(scene, cam, 0.4)
    for f in sp.dtype.names:
        if f != "pad_":
            assert np.array_equal(sp[f], _REF["splats_" + f]), f


def test_oracle_gradients_equal_reference_outputs():
    scene, cam, w = RG.case_grads()
    img, tape = O.forward_train(scene, cam, 0.6, RG.BG)
    assert np.array_equal(img, _REF["grads_img"])
    g = O.backward(scene, cam, tape, w)
    for k, v in g.items():
        b = _REF["grads_" + k]
        assert np.abs(np.asarray(v) - b).max(initial=0.0) <= 1e-12 * max(np.abs(b).max(initial=0.0), 1e-300), k
    st = O.AdamState(scene)
    for _ in range(3):
        O.optimizer_step(scene, g, st, mean_lr_scale=0.7)
    assert st.skipped_nonfinite == int(_REF["adam_skipped"])
    for f in FIELDS:
        assert np.allclose(getattr(scene, f), _REF["adam_" + f], rtol=1e-13, atol=1e-15), f


def test_oracle_sweep_equals_reference_outputs():
    s = RG.case_sweep()
    moved, rep = O.sweep_convert(s, None)
    assert np.array_equal(moved, _REF["sweep_moved"])
    assert rep["count"] == int(_REF["sweep_report"][0])
    assert abs(rep["max_leakage"] - _REF["sweep_report"][1]) <= 1e-14
    for f in FIELDS:
        assert np.allclose(getattr(s, f), _REF["sweep_" + f], rtol=0, atol=1e-14), f


def test_golden_checkpoint_is_the_reference_writers_bytes():
    """ckpt_small.hgsc equals what the reference's own save_checkpoint writes
    for the same scene and state (checked where oracle/_ref is built)."""
    from oracle import ref as R

    if not R.available():
        import pytest

        pytest.skip("oracle/_ref not built")
    import tempfile

    _sys.path.insert(0, GOLDEN)
    import make_golden as G

    s = G.golden_scene()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "ref.hgsc")
        R.save_checkpoint(s, p, G.golden_state(s))
        assert open(p, "rb").read() == open(os.path.join(GOLDEN, "ckpt_small.hgsc"), "rb").read()
