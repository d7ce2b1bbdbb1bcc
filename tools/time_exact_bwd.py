"""Times one c2 backward (K6 + exact pixels + K7b + K7) in the default mode
and in the exact backward mode (hgs_set_exact_backward), CUDA events on the
context stream."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene

ctx = Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
scene = synthetic_scene(240_000, 60_000, 3, seed=2, tau=0.5)
cam = ring_camera(2, 1352, 1014, index=0, n_ring=16)
ctx.upload(scene)
ctx.forward_train(cam, 0.0, (0.2, 0.2, 0.2))
w = np.random.default_rng(0).uniform(-1e-7, 1e-7, (1014, 1352, 3)).astype(np.float32)
wd = torch.as_tensor(w, device="cuda")
out = {}
for mode in (False, True):
    ctx.set_exact_backward(mode)
    for _ in range(2):
        ctx.backward_device(wd.data_ptr()) if hasattr(ctx, "backward_device") else ctx.backward(w)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    a.record(st)
    for _ in range(n):
        ctx.backward(w)
    b.record(st)
    torch.cuda.synchronize()
    out["exact" if mode else "default"] = a.elapsed_time(b) / n
ctx.set_exact_backward(False)
print(json.dumps({"backward_ms_incl_h2d_of_dLdimage": out}))
