"""Short run of a given config for ncu: CFG (default c2), STEPS (3) training iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.train import DeviceTrainer

scene, target, cams, times, _ = bench.workload(os.environ.get("CFG", "c2"))
ctx = Context(0)
tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2))
for i in range(int(os.environ.get("STEPS", "3"))):
    tr.step([i % len(cams)])
torch.cuda.synchronize()
print("ok", ctx.render_info())
