"""Per-phase timing of forward renders (CFG = c1 / c5 ...), CUDA events on the context stream."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13215_b200 import _capi
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene

c = CONFIGS[os.environ.get("CFG", "c5")]
scene = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"])
ctx = Context(0)
ctx.upload(scene)
cam = ring_camera(c["seed"], c["width"], c["height"], index=0, n_ring=16)
for j in range(5):
    ctx.render(cam, j / 49.0, (0.2, 0.2, 0.2))
lib = _capi.lib()
lib.hgs_profile(ctx.handle, 1)
lib.hgs_profile_read(ctx.handle, None, None, 1)
K = 20
for j in range(K):
    ctx.render(cam, j / 49.0, (0.2, 0.2, 0.2))
ph = (C.c_double * 16)()
lib.hgs_profile_read(ctx.handle, ph, None, 1)
print({n: round(ph[i] / K, 4) for i, n in enumerate(_capi.PHASES) if ph[i] > 0}, "sum", round(sum(ph) / K, 4))
print(ctx.render_info())
