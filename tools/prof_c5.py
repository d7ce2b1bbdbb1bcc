"""The bench's c5 render sweep (configs[4]: 4M Gaussians, 2048x1088,
t = j/49), small, for an ncu launch list: SWEEP frames, twice (the first
sizes the instance capacity)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene

c = CONFIGS[os.environ.get("CFG", "c5")]
n = int(os.environ.get("SWEEP", "4"))
ctx = Context(0)
ctx.upload(synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"]))
cams = [ring_camera(c["seed"], c["width"], c["height"], index=0, n_ring=16)] * n
ts = [j / 49.0 for j in range(n)]
ctx.render_sweep(cams, ts, (0.2, 0.2, 0.2))
ctx.render_sweep(cams, ts, (0.2, 0.2, 0.2))
torch.cuda.synchronize()
print("ok", ctx.render_info())
