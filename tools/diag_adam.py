import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2505_13215_b200.scene import HybridScene
from paper_2505_13215_b200.api import Context
ctx = Context(0)
rng = O.Rng(91)
scene = rng.random_scene(50, 50, 1).as_float32_exact()
cam = rng.random_camera(64, 64)
ctx.upload(scene)
st = O.AdamState(scene)
ref = scene.copy()
for it in range(3):
    ctx.forward_train(cam, 0.5, (0.2, 0.2, 0.2))
    w = np.random.default_rng(it).uniform(-1, 1, (64, 64, 3))
    if it == 1:
        w[10:14, 10:14, 0] = np.nan
    ctx.backward(w)
    g = ctx.grads()
    sk = ctx.adam_step(mean_lr_scale=0.7)
    b0 = st.skipped_nonfinite
    O.optimizer_step(ref, g, st, mean_lr_scale=0.7)
    print("it", it, "skipped", sk, st.skipped_nonfinite - b0)
    got = ctx.download(); m, v, step = ctx.adam_state()
    for f in ("mean_x", "op4", "mean3", "ql"):
        a, b = getattr(m, f), getattr(st.m, f)
        d = np.abs(a - b)
        i = np.unravel_index(np.argmax(d), d.shape)
        print(f, "max|dm|", d.max(), "at", i, "gpu", a[i], "ref", b[i], "grad", g[f][i], "p gpu", getattr(got, f)[i], "p ref", getattr(ref, f)[i])
    ref = got.copy()
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        setattr(st.m, f, getattr(m, f).copy()); setattr(st.v, f, getattr(v, f).copy())
