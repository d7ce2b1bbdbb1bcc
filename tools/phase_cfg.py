"""Per-phase CUDA-event timing of training steps for a config (CFG, default
c4) with VIEWS views per step: hgs_profile phases averaged over STEPS steps."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2505_13215_b200 import _capi
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.train import DeviceTrainer

cfg = os.environ.get("CFG", "c4")
views = int(os.environ.get("VIEWS", "8"))
steps = int(os.environ.get("STEPS", "4"))
scene, target, cams, times, _ = bench.workload(cfg)
ctx = Context(0)
tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2))
for i in range(2):
    tr.step([(i * views + j) % len(cams) for j in range(views)])
lib = _capi.lib()
lib.hgs_profile(ctx.handle, 1)
lib.hgs_profile_read(ctx.handle, None, None, 1)
for i in range(steps):
    tr.step([(i * views + j) % len(cams) for j in range(views)])
ms = (C.c_double * 16)()
calls = (C.c_longlong * 16)()
lib.hgs_profile_read(ctx.handle, ms, calls, 1)
names = list(_capi.PHASES)
tot = 0.0
for i in range(16):
    if calls[i]:
        print(f"{names[i] if i < len(names) else i:14s} {ms[i] / steps:8.3f} ms/step  calls {calls[i]}")
        tot += ms[i] / steps
print(f"sum {tot:.3f} ms/step ({views} views)", ctx.render_info())
