"""Diagnostic: per-class gradient error report at configs[1] full size and in
the dense stress scene (GPU vs the FP64 oracle).  Writes a JSON summary with
the worst elements of every class to gpurun_out/ (or argv[1])."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
from paper_2505_13215_b200.api import Context
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene
from paper_2505_13215_b200.train import quantize_8bit

CL = ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4", "mean3", "quat3", "log_s3", "op3", "sh3",
      "screen_norm4", "screen_norm3")


def report(g, r, tag):
    out = {}
    for k in CL:
        a = np.asarray(g[k], np.float64)
        b = np.asarray(r[k], np.float64)
        if a.size == 0:
            continue
        a2, b2 = a.reshape(len(a), -1), b.reshape(len(b), -1)
        e = np.abs(a2 - b2) / np.maximum(np.maximum(np.abs(a2), np.abs(b2)), 1e-6)
        bad = np.argwhere(e > 1e-3)
        rows = []
        for (i, c) in bad[np.argsort(-e[tuple(bad.T)])][:12]:
            rows.append(dict(i=int(i), c=int(c), gpu=float(a2[i, c]), ref=float(b2[i, c]), rel=float(e[i, c]),
                             row_max=float(np.abs(b2[i]).max()), cls_max=float(np.abs(b2).max())))
        ab = np.abs(b2[np.isfinite(b2)])
        out[k] = dict(n=int(e.size), n_bad=int(len(bad)), max_rel=float(e.max()),
                      n_bad_rows=int(len(np.unique(bad[:, 0]))) if len(bad) else 0,
                      q_abs=[float(np.quantile(ab, q)) for q in (0.1, 0.5, 0.9, 0.99)] if ab.size else [],
                      frac_below_floor=float((ab < 1e-6).mean()) if ab.size else 0.0,
                      err_q=[float(np.quantile(e, q)) for q in (0.5, 0.99, 0.999, 0.9999)],
                      worst=rows)
        print(tag, k, "n", e.size, "bad", len(bad), "max_rel %.3g" % e.max(), "|g| q50 %.3g" % np.median(ab),
              "below floor %.3f" % out[k]["frac_below_floor"], flush=True)
    return out


def c2(ctx):
    scene = synthetic_scene(240_000, 60_000, 3, seed=2, tau=0.5).as_float32_exact()
    target = synthetic_scene(240_000, 60_000, 3, seed=1002, tau=0.5)
    cam = ring_camera(2, 1352, 1014, index=0, n_ring=16)
    bg = (0.2, 0.2, 0.2)
    ctx.upload(target)
    gt = quantize_8bit(ctx.render(cam, 0.0, bg)["rgb"].astype(np.float64))
    ctx.upload(scene)
    img = ctx.forward_train(cam, 0.0, bg)
    loss, w = O.photometric_loss_with_grad(img.astype(np.float64), gt, 0.2)
    w = w.astype(np.float32).astype(np.float64)  # the device backward takes FP32 dL/dimage: identical inputs
    t0 = time.time()
    ref_img, tape = O.forward_train(scene, cam, 0.0, bg, num_threads=O.hardware_threads())
    print("oracle fwd s", time.time() - t0, "img err", float(np.abs(img - ref_img).max()), flush=True)
    ctx.backward(w)
    g = ctx.grads()
    t0 = time.time()
    r = O.backward(scene, cam, tape, w)
    print("oracle bwd s", time.time() - t0, flush=True)
    return report(g, r, "c2"), ctx.render_info()


def dense(ctx):
    scene = synthetic_scene(3000, 1000, 3, seed=11, density_n=100).as_float32_exact()
    cam = ring_camera(11, 160, 120)
    w = np.random.default_rng(5).uniform(-1, 1, (120, 160, 3)).astype(np.float32).astype(np.float64)
    ctx.upload(scene)
    img = ctx.forward_train(cam, 0.5, (0.2, 0.2, 0.2))
    ref, tape = O.forward_train(scene, cam, 0.5, (0.2, 0.2, 0.2), num_threads=8)
    ctx.backward(w)
    g = ctx.grads()
    r = O.backward(scene, cam, tape, w)
    return report(g, r, "dense"), ctx.render_info()


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/diag_grads.json"
    ctx = Context(0)
    res = {}
    res["dense"] = dense(ctx)
    res["c2"] = c2(ctx)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1, default=str)
