"""A few renders of config CFG (for ncu captures of the render kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene

c = CONFIGS[os.environ.get("CFG", "c5")]
scene = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"])
ctx = Context(0)
ctx.upload(scene)
cam = ring_camera(c["seed"], c["width"], c["height"], index=0, n_ring=16)
for j in range(3):
    ctx.render(cam, j / 49.0, (0.2, 0.2, 0.2))
print("ok", ctx.render_info())
