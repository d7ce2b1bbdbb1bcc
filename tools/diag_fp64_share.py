"""Share of visible splats (and of their tile instances) that take the FP64
exponent path in K4/K6 (Cholesky anisotropy r = |l01|/l11 > 4), c2 view."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2505_13215_b200.api import Context

scene, target, cams, times, _ = bench.workload(os.environ.get("CFG", "c2"))
ctx = Context(0)
ctx.upload(scene)
ctx.render(cams[0], times[0], (0.2, 0.2, 0.2))
d = ctx.debug_splats()
s = 0.5 * 1.4426950408889634
a00, a01, a11 = s * d["conic"][:, 0], s * 0.5 * (d["conic"][:, 1] + d["conic"][:, 2]), s * d["conic"][:, 3]
l00 = np.sqrt(np.maximum(a00, 1e-300))
l01 = a01 / l00
rem = a11 - l01 * l01
l11 = np.sqrt(np.maximum(rem, 1e-300))
r = np.abs(l01) / l11
fp64 = (a00 <= 0) | (rem <= 0) | (r > 4.0)
b = d["box"]
tiles = ((b[:, 1] // 16 - b[:, 0] // 16 + 1) * (b[:, 3] // 16 - b[:, 2] // 16 + 1))
print(f"visible {len(r)}  fp64 splats {fp64.mean():.3%}  fp64 share of tile instances {tiles[fp64].sum() / tiles.sum():.3%}")
print("r quantiles", np.quantile(r, [0.5, 0.9, 0.99, 0.999]))
