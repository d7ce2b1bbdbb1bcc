"""Per-step timing spread of the device-resident and host-GT (e2e) training steps."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2505_13215_b200 import _capi
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.train import DeviceTrainer

scene, target, cams, times, _ = bench.workload("c2")
ctx = Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2), iterations=1000)
for v in range(len(cams)):
    ctx.render(cams[v], times[v], (0.2, 0.2, 0.2))
lib = _capi.lib()
H, W = cams[0].height, cams[0].width
gts = [torch.empty((H, W, 3), dtype=torch.float32).pin_memory() for _ in cams]
for i, g in enumerate(gts):
    g.copy_(tr.gt[i].cpu())


def dev_step(i):
    tr.step([i % len(cams)])


def e2e_step(i):
    v = i % len(cams)
    karr = (_capi.Camera_ * 1)(tr._cams[v])
    tarr = (C.c_double * 1)(times[v])
    garr = (C.c_void_p * 1)(C.c_void_p(gts[v].data_ptr()))
    loss = C.c_double()
    tr.iter += 1
    ctx._check(lib.hgs_train_step_host(ctx.handle, 1, karr, tarr, garr, _capi.HGS_F32, 1,
                                       C.byref(tr._opts(tr.decay())), 1, C.byref(loss)))


for name, fn in (("device", dev_step), ("e2e", e2e_step), ("device", dev_step), ("e2e", e2e_step)):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    ts = []
    for i in range(60):
        t0 = time.perf_counter()
        fn(i)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts = np.array(ts)
    print(f"{name:7s} wall ms/step: median {np.median(ts):.3f} p10 {np.percentile(ts, 10):.3f} "
          f"p90 {np.percentile(ts, 90):.3f} max {ts.max():.3f}", flush=True)
