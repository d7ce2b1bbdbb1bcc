"""Writes tests/golden/ref_golden.npz: outputs of the REFERENCE itself
(oracle/_ref/libhgs_ref.so = /root/reference/proj/src compiled against
oracle/ref_shim, oracle/Makefile target ``ref``) on fixed oracle fixtures,
so the oracle stays pinned against reference-produced numbers where the
reference cannot be compiled (tests/test_golden_cpu.py).  Run once, here
(it needs /root/reference); the fixtures are committed.

Cases (scenes from oracle.Rng(seed).random_scene, as_float32_exact):
  render    -- seed 301, 60 statics + 60 dynamics, SH 3, 96x80 camera, t = 0.4,
               bg (0.1, 0.2, 0.3): rgb, count map, transmittance, RenderStats;
  splats    -- project_scene of the same scene (every splat field);
  grads     -- seed 302, 25 + 25, SH 2, 64x48, t = 0.6, loss gradient
               U(-1, 1) from numpy seed 302: forward_train image + backward;
  sweep     -- seed 303, 9 statics + 150 dynamics, SH 1, tau = 0.3:
               sweep_convert moved list and converted pools;
  adam      -- the grads case's gradients, 3 optimizer_step calls from fresh
               state (mean_lr_scale 0.7): the updated scene."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402
from paper_2505_13215_b200.scene import HybridScene  # noqa: E402

FIELDS = HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS
BG = (0.1, 0.2, 0.3)


def case_render():
    r = O.Rng(301)
    return r.random_scene(60, 60, 3).as_float32_exact(), r.random_camera(96, 80)


def case_grads():
    r = O.Rng(302)
    scene, cam = r.random_scene(25, 25, 2).as_float32_exact(), r.random_camera(64, 48)
    return scene, cam, np.random.default_rng(302).uniform(-1, 1, (48, 64, 3))


def case_sweep():
    s = O.Rng(303).random_scene(9, 150, 1).as_float32_exact()
    s.tau = 0.3
    return s


if __name__ == "__main__":
    out = {}
    scene, cam = case_render()
    r = R.rasterize(scene, cam, 0.4, BG, count_map=True, transmittance_map=True)
    out["render_rgb"], out["render_counts"], out["render_trans"] = r["rgb"], r["counts"], r["transmittance"]
    out["render_stats"] = np.array([r["stats"][k] for k in sorted(r["stats"])], np.int64)
    sp, _ = R.project_scene(scene, cam, 0.4)
    for f in sp.dtype.names:
        out["splats_" + f] = sp[f]
    scene, cam, w = case_grads()
    img, g = R.forward_backward(scene, cam, 0.6, BG, w)
    out["grads_img"] = img
    for k, v in g.items():
        out["grads_" + k] = np.asarray(v)
    a, skipped = R.optimizer_steps(scene, g, 3, mean_lr_scale=0.7)
    for f in FIELDS:
        out["adam_" + f] = getattr(a, f)
    out["adam_skipped"] = np.array(skipped)
    conv, moved, rep = R.sweep_convert(case_sweep())
    out["sweep_moved"] = moved
    out["sweep_report"] = np.array([rep["count"], rep["max_leakage"], rep["mean_leakage"]])
    for f in FIELDS:
        out["sweep_" + f] = getattr(conv, f)
    np.savez_compressed(os.path.join(HERE, "ref_golden.npz"), **out)
    print("wrote", os.path.getsize(os.path.join(HERE, "ref_golden.npz")), "bytes")
