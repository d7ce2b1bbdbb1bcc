"""Diagnostic: where do GPU gradients deviate from the oracle (dense scene)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2505_13215_b200.scene import synthetic_scene, ring_camera
from paper_2505_13215_b200.api import Context

ctx = Context(0)
scene = synthetic_scene(3000, 1000, 3, seed=11, density_n=100).as_float32_exact()
cam = ring_camera(11, 160, 120)
w = np.random.default_rng(5).uniform(-1, 1, (120, 160, 3))
ctx.upload(scene)
img = ctx.forward_train(cam, 0.5, (0.2, 0.2, 0.2))
print("render info", ctx.render_info())
ref, tape = O.forward_train(scene, cam, 0.5, (0.2, 0.2, 0.2), num_threads=8)
print("img err", np.abs(img - ref).max())
ctx.backward(w)
g = ctx.grads()
r = O.backward(scene, cam, tape, w)
for k in ("mean_x", "op4", "sh4", "log_s4", "mean3", "op3", "screen_norm4"):
    a, b = g[k].reshape(len(g[k]), -1), r[k].reshape(len(r[k]), -1)
    e = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-6)
    bad = np.argwhere(e > 1e-3)
    print(k, "bad", len(bad), "of", e.size, "max abs err", np.abs(a - b).max(), "max |g|", np.abs(b).max())
    for (i, c) in bad[np.argsort(-e[tuple(bad.T)])][:6]:
        print("   ", i, c, "gpu", a[i, c], "ref", b[i, c], "rel", e[i, c], "row max", np.abs(b[i]).max())
print("--- scale-normalised (floor = 1e-6 * max|g| per class)")
for k in ("mean_x", "mean_t", "ql", "qr", "op4", "sh4", "log_s4", "mean3", "quat3", "log_s3", "op3", "sh3"):
    a, b = g[k].ravel(), r[k].ravel()
    fl = max(1e-6, 1e-6 * np.abs(b).max())
    e = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), fl)
    print(k, "frac>1e-3", (e > 1e-3).mean(), "max", e.max())
