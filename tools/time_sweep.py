"""ms per frame of the bench's render sweep for a config (CFG, default c5;
FRAMES frames per sweep, REPS timed sweeps): quick A/B of render-path changes
(HGS_LIB selects the library)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene

name = os.environ.get("CFG", "c5")
c = CONFIGS[name]
k = int(os.environ.get("FRAMES", "20"))
reps = int(os.environ.get("REPS", "3"))
ctx = Context(0)
ctx.upload(synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"]))
cams = [ring_camera(c["seed"], c["width"], c["height"], index=0, n_ring=16)] * k
ts = [(j % 50) / 49.0 for j in range(k)] if name == "c5" else [c["t"]] * k
ctx.render_sweep(cams, ts, (0.2, 0.2, 0.2))
best = 1e30
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.render_sweep(cams, ts, (0.2, 0.2, 0.2))
    torch.cuda.synchronize()
    best = min(best, (time.perf_counter() - t0) * 1e3 / k)
print(f"{os.environ.get('HGS_LIB', 'default')} {name} ms/frame {best:.4f} Mpix/s {c['width'] * c['height'] / best / 1e3:.1f}")
