"""A small end-to-end run (the checked-build workload, tests/test_gpu_checked.py) of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): render (full instance list
and the fused production path), render sweep with a forced capacity overflow,
forward_train / loss / backward (default and exact mode), Adam, train steps
(sync + pipelined), sweep, densify, density map, checkpoint save/load."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2505_13215_b200.api import Context, Rng
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene
from paper_2505_13215_b200.train import DeviceTrainer

# HGS_RUN_SCALE=k: k times the Gaussians and k times the image side (checked-build test)
k = int(os.environ.get("HGS_RUN_SCALE", "1"))
ctx = Context(0)
scene = synthetic_scene(1500 * k, 800 * k, 2, seed=5, density_n=1500 * k)
target = synthetic_scene(1500 * k, 800 * k, 2, seed=6, density_n=1500 * k)
cams = [ring_camera(5, 96 * k, 72 * k, index=i, n_ring=4) for i in range(4)]
bg = (0.2, 0.2, 0.2)
ctx.upload(scene)
ctx.render(cams[0], 0.5, bg)
ctx._lib.hgs_debug_keep_instances(ctx.handle, 1)
ctx.render(cams[1], 0.3, bg, count_map=True, transmittance_map=True)
ctx._lib.hgs_debug_keep_instances(ctx.handle, 0)
ctx.render_sweep([cams[2]] * 6, [j / 5 for j in range(6)], bg)
w = np.random.default_rng(0).uniform(-1, 1, (72 * k, 96 * k, 3))
for exact in (False, True):
    ctx.set_exact_backward(exact)
    ctx.forward_train(cams[0], 0.5, bg)
    ctx.backward(w)
ctx.set_exact_backward(False)
ctx.adam_step()
tr = DeviceTrainer(ctx, scene, cams, [0.1, 0.4, 0.6, 0.9], target=target, bg=bg, iterations=20)
for i in range(3):
    tr.step([i % 4, (i + 1) % 4])
for i in range(3):
    tr.step_async([i % 4, (i + 2) % 4])
while ctx._lib.hgs_train_pending(ctx.handle):
    tr.collect()
ctx.sweep_convert()
ctx.densify_and_prune(Rng(3), grad_threshold=1e-7, max_gaussians=5000)
ctx.density_map(cams[0], 0.5)
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "s.hgsc")
    ctx.save_checkpoint(p)
    ctx.load_checkpoint(p)
ctx.synchronize()
print("sanitize run ok")
