"""The rasterizers' tile launch order (heaviest tiles first, tile_order_kernel)
and the in-CTA FP64 fix-up do not change any result: a render with the order
disabled (HGS_NO_TILE_ORDER=1, read once per process) gives the same image,
transmittance, last-contributor map and fix-up pixel count bit for bit."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import hashlib, sys
sys.path.insert(0, sys.argv[1])
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene
ctx = Context(0)
ctx.upload(synthetic_scene(60000, 20000, 3, seed=21))
h = hashlib.sha256()
for i in range(3):
    out = ctx.render(ring_camera(21, 640, 480, index=i, n_ring=3), 0.3 * i, (0.2, 0.2, 0.2), transmittance_map=True)
    h.update(out["rgb"].tobytes())
    h.update(out["transmittance"].tobytes())
    h.update(str(ctx.render_info()).encode())
print("HASH", h.hexdigest())
'''


@pytest.mark.gpu
def test_tile_launch_order_does_not_change_results():
    hashes = []
    for order_off in ("0", "1"):
        env = dict(os.environ)
        env.pop("HGS_NO_TILE_ORDER", None)
        if order_off == "1":
            env["HGS_NO_TILE_ORDER"] = "1"
        r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        hashes.append([l for l in r.stdout.splitlines() if l.startswith("HASH")][0])
    assert hashes[0] == hashes[1]
