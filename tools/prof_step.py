"""Short c2 run for ncu: 2 warm-up training iterations + 1 profiled one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.train import DeviceTrainer
import bench

scene, target, cams, times, _ = bench.workload(os.environ.get("CFG", "c2"))
ctx = Context(0)
tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2))
n = int(os.environ.get("STEPS", "3"))
for i in range(n):
    tr.step([i % len(cams)])
torch.cuda.synchronize()
print("ok", ctx.render_info())
