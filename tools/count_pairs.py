"""Pixel-splat pair counts of the tile rasterizers on the c2 training step
(the checked build's counters, hgs_debug_pair_counters): for K4 and K6 the
lane-iterations, the box-covered pairs whose exponent is evaluated (E), the
alpha-passing pairs that are composited / back-propagated, and the
warp-iterations.  Writes profiles/<tag>_pairs.json (read by bench.py's
roofline).  Run on the GPU box:
  HGS_LIB=paper_2505_13215_b200/libhgs_gpu_checked.so python tools/count_pairs.py r02"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HGS_LIB", os.path.join(ROOT, "paper_2505_13215_b200", "libhgs_gpu_checked.so"))
import bench
from paper_2505_13215_b200 import _capi
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.train import DeviceTrainer

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
cfg = os.environ.get("CFG", "c2")
scene, target, cams, times, desc = bench.workload(cfg)
ctx = Context(0)
tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2))
lib = _capi.lib()
out = (C.c_ulonglong * 8)()
tr.step([0])
ctx.synchronize()
assert lib.hgs_debug_pair_counters(ctx.handle, out, 1) == 0, "needs the checked build"
views = 4
tot = [0] * 8
for v in range(views):
    tr.step([v % len(cams)])
    ctx.synchronize()
    lib.hgs_debug_pair_counters(ctx.handle, out, 1)
    tot = [a + b for a, b in zip(tot, out)]
per = [t / views for t in tot]
names = ["lane_iterations", "box_pairs_evaluated", "alpha_passing_pairs", "warp_iterations"]
res = {"config": cfg, "views_averaged": views, "library": os.path.basename(os.environ["HGS_LIB"]),
       "what": "per training iteration (one view): box pairs = (pixel, splat) pairs whose exponent K4/K6 evaluate; "
               "alpha-passing = pairs composited (K4) / back-propagated (K6); lane/warp iterations of the splat walks",
       "raster_fwd": dict(zip(names, per[:4])), "raster_bwd": dict(zip(names, per[4:]))}
for k in ("raster_fwd", "raster_bwd"):
    d = res[k]
    d["pass_fraction"] = d["alpha_passing_pairs"] / max(1.0, d["box_pairs_evaluated"])
    d["pairs_per_warp_iteration"] = d["box_pairs_evaluated"] / max(1.0, d["warp_iterations"])
path = os.path.join(ROOT, "profiles", f"{tag}_pairs.json")
json.dump(res, open(path, "w"), indent=1)
print(json.dumps(res, indent=1))
