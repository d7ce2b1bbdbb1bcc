"""Experiment: fraction of box-covered / alpha-passing pixel pairs per warp iteration of K4."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2505_13215_b200 import _capi
from paper_2505_13215_b200.api import Context

scene, target, cams, times, _ = bench.workload("c2")
ctx = Context(0)
ctx.upload(scene)
lib = _capi.lib()
f = lib.hgs_exp_counters
f.argtypes = [C.POINTER(C.c_ulonglong)]
out = (C.c_ulonglong * 4)()
ctx.render(cams[0], times[0], (0.2, 0.2, 0.2))
f(out)
ctx.render(cams[0], times[0], (0.2, 0.2, 0.2))
f(out)
w, b, p = out[0], out[1], out[2]
print(f"warp-iterations {w}, box pairs {b} ({b / (64 * w):.3f} of 64 px), alpha-passing pairs {p} ({p / (64 * w):.3f})")
print(ctx.render_info())
