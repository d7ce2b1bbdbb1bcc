#!/usr/bin/env python
"""bench.py -- throughput of the hybrid 3D/4DGS training hot path on B200.

Default workload (BASELINE.json configs[1], "c2"): 240k 4D + 60k 3D Gaussians,
SH degree 3, 1352x1014, one training view per GPU per iteration (slice +
projection + SH, sorts, tile rasterizer forward, L1 + D-SSIM loss, rasterizer
backward, per-Gaussian backward, fused Adam).  Synthetic data: the scene and
the ground-truth scene (seed + 1000, rendered once on the GPU and 8-bit
quantised like the reference's generate_synthetic) follow SURVEY.md 8d.

  python bench.py [--gpus N --steps K --warmup W]            # this repo (CUDA)
  python bench.py --impl reference [...]                      # CPU reference path

One JSON line on rank 0.  value = views/s over all ranks (one view = one
training iteration of one 1352x1014 camera; weak scaling: N GPUs -> N views
per iteration + one NCCL all-reduce of the packed gradients).  The working
set (params + Adam moments + grads ~ 0.3 GB) exceeds the 126 MB L2, so no
explicit flush is needed between iterations.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "views/s"
HBM_FALLBACK_GBS = 6650.0


def peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


# ------------------------------------------------------------------ workload
def workload(cfg_name: str):
    from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene

    c = CONFIGS[cfg_name]
    n4, n3, W, H, seed = c["n4"], c["n3"], c["width"], c["height"], c["seed"]
    scene = synthetic_scene(n4, n3, 3, seed=seed, tau=0.5)
    target = synthetic_scene(n4, n3, 3, seed=seed + 1000, tau=0.5)
    cams = [ring_camera(seed, W, H, index=i, n_ring=16) for i in range(16)]
    times = [i / 15.0 for i in range(16)]
    desc = {"workload": f"{cfg_name}: {n4 // 1000}k 4D + {n3 // 1000}k 3D Gaussians, SH deg 3, {W}x{H}, "
                        "1 view/GPU/iteration: slice+EWA+SH, depth+tile radix sorts, tile raster fwd, "
                        "L1+D-SSIM, raster bwd, per-Gaussian bwd, fused Adam",
            "gaussians": n4 + n3, "width": W, "height": H, "sh_degree": 3, "views_in_ring": 16,
            "l2": "working set > 126 MB L2 (no flush needed)"}
    return scene, target, cams, times, desc


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled through NVML every
    5 ms during the timed region (plus one sample at each edge, so even a
    short region is covered)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.h, self.err = gpu, [], None, None
        self.stop = threading.Event()

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        except Exception:
            bus = None
        if bus is not None:
            try:
                return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                pass
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
        return pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((sm, mx, rs))

    def _loop(self):
        while not self.stop.wait(0.005):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        try:
            self.h = self._handle()
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception as e:  # NVML missing: reported, never fatal
            self.h, self.err = None, f"nvml unavailable: {type(e).__name__}"
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        reasons = sorted({name for _, _, r in self.rows for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                "sm_max_mhz": float(max(r[1] for r in self.rows)), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


# ------------------------------------------------------------------ roofline
def algorithmic_bytes(phase: str, n: dict) -> float | None:
    """Per-step algorithmic bytes of each kernel phase (SURVEY.md 8d table,
    adapted to this implementation's passes)."""
    N4, N3, V, I, K, px, P = n["n4"], n["n3"], n["V"], n["I"], n["K"], n["px"], n["rows_avg"]
    if phase == "preprocess":   # params in (68/44 B geometry + 192 B SH of visible), 80 B record + 64 B
        return 68 * N4 + 44 * N3 + (192 + 80 + 64) * V + 4 * (N4 + N3) * 3  # colour record out, flags
    if phase == "depth_sort":   # global LSD over V keys+values: (8 + 24*passes) * n
        return (8 + 24 * 4) * V
    if phase == "duplicate":    # gather (80 B in, 80+64+8 B out) + offsets scan; 12 B per instance out
        return (80 + 152 + 12) * V + 12 * I
    if phase == "tile_sort":    # keep-flag scan (8 B per instance), compaction (8 B in per instance,
        return 16 * I + 8 * K + (8 + 16 * 2) * K  # 8 B out per kept one), 2 passes over the kept pairs
    if phase == "raster_fwd":   # K4: 4 B value + 64 B splat per kept instance, 24 B per pixel out
        return 68 * K + 24 * px
    if phase == "loss":
        return 44 * px * 3
    if phase == "raster_bwd":   # 68 B per kept instance + 36 B accumulators, 32 B per pixel in
        return 104 * K + 32 * px
    if phase == "gaussian_bwd":  # read params + write grads (2 * 4 * P) + 36 B accumulators
        return V * (2 * 4 * P + 48)
    if phase == "adam":          # 32 B per element (param, m, v rw; grad read + zero)
        return 32 * (N4 * n["rows4"] + N3 * n["rows3"])
    return None


def roofline(phase_ms: dict, counts: dict, steps: int, peak: float, peak_kind: str) -> dict:
    kernels = []
    for ph, ms in phase_ms.items():
        if ms <= 0:
            continue
        b = algorithmic_bytes(ph, counts)
        per = ms / steps
        gbs = (b / (per * 1e-3) / 1e9) if b else None
        kernels.append({"phase": ph, "ms_per_step": round(per, 4), "alg_bytes": b,
                        "GB/s": round(gbs, 1) if gbs else None, "frac": round(gbs / peak, 4) if gbs else None})
    kernels.sort(key=lambda k: -k["ms_per_step"])
    if not kernels:
        return {"bound": "hbm", "kernel": None, "achieved": None, "peak": peak, "unit": "GB/s", "frac": None,
                "traffic": None, "peak_source": peak_kind, "kernels": []}
    top = kernels[0]
    # DRAM traffic per launch of the phase's main kernel from the committed
    # `ncu --set full` capture (profiles/ncu_summary.json, tools/make_profiles.py)
    ncu = {}
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    except Exception:
        pass
    main_kernel = {"raster_bwd": "raster_bwd_kernel", "raster_fwd": "raster_fwd_kernel",
                   "duplicate": "duplicate_compact_kernel", "gaussian_bwd": "gaussian_bwd_kernel",
                   "adam": "adam_rows_kernel", "tile_sort": "radix_sort_coop_kernel",
                   "depth_sort": "radix_sort_coop_kernel", "preprocess": "preprocess_kernel",
                   "loss": "ssim_fwd_kernel"}
    for k in kernels:
        prof = ncu.get(main_kernel.get(k["phase"], ""), {})
        k["ncu"] = {key: prof.get(key) for key in ("kernel", "duration_us", "dram_bytes_per_launch",
                                                   "issue_slots_busy_pct", "ipc_active", "pipes_pct",
                                                   "report")} if prof else None
    # the rasterizers' own roofline: instruction issue.  Pixel-splat pairs per
    # step from the checked build's counters (profiles/*_pairs.json,
    # tools/count_pairs.py: a property of the workload), pipe utilisation from
    # the committed ncu capture of the kernel
    pairs = {}
    try:
        pf = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_pairs.json"))
        pairs = json.load(open(os.path.join(ROOT, "profiles", pf[-1]))) if pf else {}
        pairs["file"] = pf[-1] if pf else None
    except Exception:
        pairs = {}
    issue = {}
    for k in kernels:
        if k["phase"] in ("raster_fwd", "raster_bwd"):
            pc = pairs.get(k["phase"]) or {}
            e = pc.get("box_pairs_evaluated")
            ip = ((k.get("ncu") or {}).get("pipes_pct") or {})
            issue[k["phase"]] = {
                "bound": "instruction issue (FP32 / ALU / shared-memory pipes)",
                "issue_pct": ip.get("issue"), "fma_pipe_pct": ip.get("fma"), "alu_pipe_pct": ip.get("alu"),
                "lsu_pipe_pct": ip.get("lsu"), "xu_pipe_pct": ip.get("xu"),
                "shared_wavefront_pct": ip.get("shared_wavefronts"),
                "pairs_evaluated_per_step": e, "alpha_passing_pairs_per_step": pc.get("alpha_passing_pairs"),
                "Gpairs_per_s": round(e / (k["ms_per_step"] * 1e-3) / 1e9, 2) if e else None,
                "pairs_source": pairs.get("file"), "pipes_source": (k.get("ncu") or {}).get("report")}
    tp = (top.get("ncu") or {})
    return {"bound": "hbm", "kernel": top["phase"], "achieved": top["GB/s"], "peak": peak, "unit": "GB/s",
            "frac": top["frac"], "traffic": tp.get("dram_bytes_per_launch"), "peak_source": peak_kind,
            "note": "the tile rasterizers are issue-bound, not HBM-bound (their splat reads hit L2): "
                    "their roofline is `issue` (pipe utilisation and pixel-splat pairs per second)",
            "issue": issue, "kernels": kernels}


# ------------------------------------------------------------------ our arm
def run_ours(args) -> None:
    import torch

    from paper_2505_13215_b200 import _capi
    from paper_2505_13215_b200.api import Context
    from paper_2505_13215_b200.train import DeviceTrainer, ViewParallelTrainer, quantize_8bit

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    vp = world > 1 or args.view_parallel  # the view-parallel code path (also at N=1 with --view-parallel)
    if vp:
        import torch.distributed as dist

        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29631")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    scene, target, cams, times, desc = workload(args.config)
    ctx = Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    kw = dict(target=target, bg=(0.2, 0.2, 0.2), iterations=max(1000, args.steps * 10))
    tr = (ViewParallelTrainer(ctx, scene, cams, times, exchange="capi", sharded=args.sharded, **kw) if vp
          else DeviceTrainer(ctx, scene, cams, times, **kw))

    def batch(step):
        return [(step * world + r) % len(cams) for r in range(world)]

    # setup: one forward pass over every view sizes the device workspaces
    # (no cudaMalloc inside the timed region)
    for v in range(len(cams)):
        ctx.render(cams[v], times[v], (0.2, 0.2, 0.2))

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k, drain=None):
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(k):
            fn(i)
        if drain:
            drain()
        t1.record(stream)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        if dist:
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        barrier()
        return ms

    # Pipelined iterations (hgs_train_step_async): iteration i is enqueued
    # before iteration i-1's loss is read back (hgs_train_collect), every loss
    # is read inside the timed region.  N GPUs: the same, each rank's view
    # followed by hgs_train_exchange_async (NCCL all-reduce of the loss gate
    # and the packed gradients, gated Adam) -- no host synchronisation.
    def pending():
        return lib.hgs_train_pending(ctx.handle)

    def drain():
        while pending():
            tr.collect()

    def step_1gpu(i, gt_host=None):
        v = batch(i)[0]
        tr.step_async([v], gt_host=None if gt_host is None else [gt_host[v]])
        if pending() > 1:
            tr.collect()

    def step_ngpu(i, gt_host=None):
        b = batch(i)
        tr.step_async(b, gt_host=None if gt_host is None else [gt_host[b[rank]]])
        if pending() > 1:
            tr.collect()

    lib = _capi.lib()
    step_fn = step_ngpu if vp else step_1gpu
    for i in range(args.warmup):
        step_fn(i)
    drain()
    # ---- device-resident timed region (the headline; no instrumentation)
    l0 = _capi.lib().hgs_launch_count()
    with ClockSampler(local) as clk:
        # NVTX range "timed": `ncu --nvtx --nvtx-include timed/` lists exactly these launches
        torch.cuda.nvtx.range_push("timed")
        ms = timed(lambda i: step_fn(args.warmup + i), args.steps, drain)
        torch.cuda.nvtx.range_pop()
    launches = _capi.lib().hgs_launch_count() - l0
    import ctypes as C

    # ---- the same steps again with per-phase CUDA events (roofline.kernels);
    # the events cost ~4% of the step, so they are kept out of the headline
    phase_ms = {}
    if not args.no_phase_profile:
        _capi.lib().hgs_profile(ctx.handle, 1)
        _capi.lib().hgs_profile_read(ctx.handle, None, None, 1)
        timed(lambda i: step_fn(args.warmup + args.steps + i), args.steps, drain)
        ph = (C.c_double * 16)()
        _capi.lib().hgs_profile_read(ctx.handle, ph, None, 1)
        _capi.lib().hgs_profile(ctx.handle, 0)
        phase_ms = {name: float(ph[i]) for i, name in enumerate(_capi.PHASES)}
    info = ctx.render_info()
    value = world * args.steps / (ms / 1e3)

    # ---- end to end through the C ABI with HOST ground truth (pinned): the
    # frames as the reference's dataset holds them, 8-bit sRGB (read_ppm),
    # decoded on the device inside the loss (HGS_U8)
    from paper_2505_13215_b200.train import linear_to_srgb8

    H, W = cams[0].height, cams[0].width
    gts_host = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(len(cams))]
    for i, g in enumerate(gts_host):
        g.copy_(torch.as_tensor(linear_to_srgb8(tr.gt[i].cpu().numpy().astype(np.float64))))
    lib = _capi.lib()

    def e2e_step(i):  # pipelined like the device loop, host GT frames
        step_fn(args.warmup + args.steps + i, gt_host=gts_host)

    for i in range(args.warmup):  # untimed: the copy stream and GT buffers are created on first use
        e2e_step(-1 - i)
    drain()
    e2e_ms = timed(e2e_step, args.steps, drain)
    e2e_value = world * args.steps / (e2e_ms / 1e3)

    # ---- forward-only render throughput (Mpix/s), device resident: one
    # hgs_render_sweep of K frames (no host round trip between frames)
    sweep_cams = [cams[(i * world + rank) % len(cams)] for i in range(args.steps)]
    sweep_ts = [times[(i * world + rank) % len(cams)] for i in range(args.steps)]
    ctx.render_sweep(sweep_cams, sweep_ts, (0.2, 0.2, 0.2))  # learns the instance capacity (untimed)
    r_ms = timed(lambda _i: ctx.render_sweep(sweep_cams, sweep_ts, (0.2, 0.2, 0.2)), 1)
    render_mpix = world * args.steps * W * H / (r_ms / 1e3) / 1e6

    peak, peak_kind = peaks()
    rows4 = 17 + 48
    rows3 = 11 + 48
    counts = {"n4": scene.n4, "n3": scene.n3, "V": info["visible"], "I": info["instances"],
              "K": info["kept_instances"], "px": W * H,
              "rows4": rows4, "rows3": rows3,
              "rows_avg": (rows4 * scene.n4 + rows3 * scene.n3) / max(1, scene.n4 + scene.n3)}
    rl = roofline(phase_ms, counts, args.steps, peak, peak_kind)

    extra = run_extras(args, ctx, lib, timed, world, rank) if not args.no_extras else None
    if extra is not None and world == 1:
        extra["c3_train"] = run_c3(ctx, timed)
        extra["rows_8f"] = run_rows(ctx)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(scene, cams[0], times[0], quantize_8bit(tr.gt[0].cpu().numpy().astype(np.float64)))

    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32 (geometry, keys and guard-band decisions f64)",
               "data": "synthetic (SURVEY.md 8d generator; random init, GT = 8-bit render of a second scene)",
               "config": dict(desc, parallelism=f"view-parallel dp{world}", views_per_iteration=world),
               "e2e": {"value": round(e2e_value, 3), "unit": UNIT,
                       "h2d_bytes_per_step": int(W * H * 3),  # one 8-bit sRGB frame
                       "d2h_bytes_per_step": 16 if not vp else 24,  # loss sums (+ the all-reduced gate)
                       "path": ("hgs_train_step_async with a host 8-bit sRGB GT frame + hgs_train_collect "
                                "(pinned host frame in, loss out, every iteration)") if not vp else
                               ("hgs_train_step_async (pinned host 8-bit GT frame) + hgs_train_exchange_async "
                                "(NCCL all-reduce, gated Adam) + hgs_train_collect")},
               "render": {"value": round(render_mpix, 2), "unit": "Mpix/s",
                          "what": "forward render of the device-resident c2 scene, 1352x1014 (hgs_render_sweep "
                                  "of K frames, one synchronisation)"},
               "gpu_launches": int(launches), "launches_per_step": round(launches / args.steps, 1),
               "roofline": rl, "clocks": clk.summary(), "cpu_baseline": cpu,
               "render_info": info, "extra": extra}
        print(json.dumps(out), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


def run_extras(args, ctx, lib, timed, world, rank) -> dict:
    """The other SURVEY.md 8d configurations, measured the same way (CUDA
    events on the context stream, W untimed + K timed steps, max over ranks):
      c1 / c5: forward render throughput (Mpix/s) -- c5 is the render sweep
               (4M Gaussians, 2048x1088, t = j/49);
      c4:      training with 8 views per GPU per step (2M Gaussians)."""
    import ctypes as C

    import torch

    from paper_2505_13215_b200 import _capi
    from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene
    from paper_2505_13215_b200.train import DeviceTrainer

    out = {}
    bg = (C.c_double * 3)(0.2, 0.2, 0.2)
    for name in ("c1", "c5"):
        c = CONFIGS[name]
        scene = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"])
        ctx.upload(scene)
        ts = [j / 49.0 for j in range(50)] if name == "c5" else [c["t"]]

        k = max(args.steps, 10) * (5 if name == "c1" else 1)  # c1 frames are short: more of them
        cam_objs = [ring_camera(c["seed"], c["width"], c["height"], index=0, n_ring=16)] * k
        sweep_ts = [ts[(i * world + rank) % len(ts)] for i in range(k)]
        ctx.render_sweep(cam_objs, sweep_ts, (0.2, 0.2, 0.2))  # sizes the workspaces and the capacity (untimed)
        ms = timed(lambda _i: ctx.render_sweep(cam_objs, sweep_ts, (0.2, 0.2, 0.2)), 1)
        out[f"{name}_render"] = {"value": round(world * k * c["width"] * c["height"] / (ms / 1e3) / 1e6, 2),
                                 "unit": "Mpix/s", "ms_per_frame": round(ms / k, 4),
                                 "config": f"{c['n4'] // 1000}k 4D + {c['n3'] // 1000}k 3D, "
                                           f"{c['width']}x{c['height']}" + (", t=j/49" if name == "c5" else "")}
        del scene
    # c4: 8 views per optimizer step in TOTAL (BASELINE configs[3]), split
    # over the ranks (strong scaling of the step); at N > 1 the packed
    # gradient all-reduce + gated Adam are inside the timed region
    # (ViewParallelTrainer, hgs_train_exchange_async)
    import torch.distributed as tdist

    from paper_2505_13215_b200.train import ViewParallelTrainer

    c = CONFIGS["c4"]
    scene = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"], tau=0.5)
    target = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"] + 1000, tau=0.5)
    cams = [ring_camera(c["seed"], c["width"], c["height"], index=i, n_ring=16) for i in range(16)]
    times = [i / 15.0 for i in range(16)]
    vp = tdist.is_available() and tdist.is_initialized()
    kw = dict(target=target, bg=(0.2, 0.2, 0.2), iterations=1000)
    tr = (ViewParallelTrainer(ctx, scene, cams, times, exchange="capi", **kw) if vp
          else DeviceTrainer(ctx, scene, cams, times, **kw))
    del target
    for v in range(16):
        ctx.render(cams[v], times[v], (0.2, 0.2, 0.2))
    per_step = 8

    def step(i):
        tr.step_async([(i * per_step + j) % 16 for j in range(per_step)])
        if ctx._lib.hgs_train_pending(ctx.handle) > 1:
            tr.collect()

    def drain():
        while ctx._lib.hgs_train_pending(ctx.handle):
            tr.collect()

    for i in range(args.warmup):
        step(i)
    drain()
    k = max(2, args.steps // 2)
    ms = timed(step, k, drain)
    out["c4_train"] = {"value": round(k * per_step / (ms / 1e3), 3), "unit": "views/s",
                       "ms_per_step": round(ms / k, 4), "views_per_step": per_step,
                       "views_per_gpu_per_step": per_step / world, "scaling": "strong",
                       "exchange": "NCCL all-reduce of the packed gradients + gated Adam (timed)" if vp else "none (1 GPU)",
                       "config": "1600k 4D + 400k 3D, SH 3, 1352x1014, 8 views per optimizer step over all GPUs"}
    torch.cuda.synchronize()
    return out


def run_c3(ctx, timed) -> dict:
    """configs[2], N3V-shaped: 300k Gaussians (all 4D at start), 18 cameras x
    300 frames (t = j/299), 1352x1014, batch 2, the periodic 4D->3D conversion
    sweep every 100 iterations (train.cpp:466-472) inside the timed region.
    The 5400 8-bit GT frames (22 GB, device resident) are renders of a second
    scene, encoded on the device (render_gt_u8_device)."""
    import torch

    from paper_2505_13215_b200.rng import MT19937_64, uniform_index
    from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene
    from paper_2505_13215_b200.train import DeviceTrainer, render_gt_u8_device

    c = CONFIGS["c3"]
    scene = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"], tau=0.5)
    target = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"] + 1000, tau=0.5)
    cams, times = [], []
    for ci in range(18):
        cam = ring_camera(c["seed"], c["width"], c["height"], index=ci, n_ring=18)
        for j in range(300):
            cams.append(cam)
            times.append(j / 299.0)
    gts = render_gt_u8_device(ctx, target, cams, times, bg=(0.2, 0.2, 0.2))
    tr = DeviceTrainer(ctx, scene, cams, times, bg=(0.2, 0.2, 0.2), iterations=400, gt_format="u8", gt_device=gts)
    del target
    rng = MT19937_64(3)
    n = len(cams)
    state = {"it": 0, "moved": 0, "sweeps": 0}

    def iteration(_):
        state["it"] += 1
        tr.step_async([uniform_index(rng, 0, n - 1) for _ in range(2)])
        if ctx._lib.hgs_train_pending(ctx.handle) > 1:
            tr.collect()
        if state["it"] % 100 == 0:  # drain, then the sweep (train.cpp:466-472)
            while ctx._lib.hgs_train_pending(ctx.handle):
                tr.collect()
            moved, _ = ctx.sweep_convert()
            state["moved"] += len(moved)
            state["sweeps"] += 1

    def drain():
        while ctx._lib.hgs_train_pending(ctx.handle):
            tr.collect()

    for i in range(20):  # warm-up (no sweep)
        tr.step_async([uniform_index(rng, 0, n - 1) for _ in range(2)])
        tr.collect()
    state["it"] = 0
    k = 200
    ms = timed(iteration, k, drain)
    n4, n3 = ctx.counts()
    torch.cuda.synchronize()
    return {"value": round(2 * k / (ms / 1e3), 2), "unit": "views/s", "iters_per_s": round(k / (ms / 1e3), 2),
            "ms_per_iter": round(ms / k, 4), "sweeps": state["sweeps"], "converted": state["moved"],
            "final_n4": n4, "final_n3": n3,
            "config": "300k 4D (+ converted 3D), SH 3, 1352x1014, 18 cameras x 300 frames (8-bit GT, device "
                      "resident), batch 2, 4D->3D sweep every 100 iterations (timed)"}


def run_rows(ctx) -> dict:
    """The SURVEY.md 8f rows, each through its public API call at c2 scale
    (host-synchronous calls: wall time around the call, synchronised on both
    sides -- these are end-to-end numbers including their host work)."""
    import tempfile

    import torch

    from paper_2505_13215_b200 import api as A
    from paper_2505_13215_b200 import dataset as D
    from paper_2505_13215_b200.scene import CONFIGS, ring_camera, synthetic_scene
    from paper_2505_13215_b200.train import DeviceTrainer

    def wall(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3, r

    out = {}
    c = CONFIGS["c2"]
    scene = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"], tau=0.5)
    target = synthetic_scene(c["n4"], c["n3"], 3, seed=c["seed"] + 1000, tau=0.5)
    cams = [ring_camera(c["seed"], c["width"], c["height"], index=i, n_ring=16) for i in range(16)]
    times = [i / 15.0 for i in range(16)]
    tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2), iterations=1000, gt_format="u8")
    del target
    for i in range(8):
        tr.step([(2 * i) % 16, (2 * i + 1) % 16])
    n_before = sum(ctx.counts())
    gn4, c4, gn3, c3 = ctx.densify_stats()
    avg = np.concatenate([gn4 / np.maximum(c4, 1), gn3 / np.maximum(c3, 1)])
    thr = float(np.quantile(avg[avg > 0], 0.98)) if (avg > 0).any() else 0.02  # ~2% of the observed densify
    ms, rep = wall(lambda: ctx.densify_and_prune(A.Rng(7), grad_threshold=thr, max_gaussians=1_000_000))
    out["densify_and_prune"] = {"ms": round(ms, 3), "gaussians_before": n_before, "gaussians_after": sum(ctx.counts()),
                                "report": rep, "grad_threshold": thr,
                                "what": "hgs_densify_and_prune: device plan + libstdc++ normal draws + device apply"}
    frames = [t.cpu().numpy() for t in tr.gt]  # host u8 sRGB frames
    for v in range(2):
        ctx.render_device(cams[v], times[v], (0.2, 0.2, 0.2))
        ctx.image_metrics(frames[v])

    def evaluate():
        for v in range(16):
            ctx.render_device(cams[v], times[v], (0.2, 0.2, 0.2))
            ctx.image_metrics(frames[v])

    ms, _ = wall(evaluate)
    out["evaluate_views"] = {"value": round(16 / (ms / 1e3), 2), "unit": "views/s", "ms_per_view": round(ms / 16, 4),
                             "what": "render (no download) + PSNR + SSIM vs a host u8 frame, c2 scene 1352x1014"}
    ctx.density_map(cams[0], 0.5)
    ms, _ = wall(lambda: [ctx.density_map(cams[v], times[v]) for v in range(8)])
    out["density_map"] = {"ms_per_map": round(ms / 8, 4), "what": "c2 scene, 1352x1014 counts downloaded"}
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "c2.hgsc")
        ctx.save_checkpoint(p)
        ms_s, _ = wall(lambda: ctx.save_checkpoint(p))
        size = os.path.getsize(p)
        ms_l, _ = wall(lambda: ctx.load_checkpoint(p))
        out["checkpoint"] = {"bytes": size, "save_ms": round(ms_s, 2), "load_ms": round(ms_l, 2),
                             "save_GBps": round(size / ms_s / 1e6, 2), "load_GBps": round(size / ms_l / 1e6, 2),
                             "what": "device scene + optimizer state <-> .hgsc file (page cache), CRC-32 included"}
        w, h = c["width"], c["height"]
        rng = np.random.default_rng(0)
        paths = []
        for i in range(32):
            paths.append(os.path.join(d, f"f{i}.ppm"))
            D.write_ppm(rng.integers(0, 256, (h, w, 3), dtype=np.uint8), paths[-1])
        buf = torch.empty((32, h, w, 3), dtype=torch.uint8).pin_memory().numpy()
        D.read_ppm_batch(paths, w, h, out=buf)
        ms, _ = wall(lambda: D.read_ppm_batch(paths, w, h, out=buf))
        out["ppm_read_batch"] = {"value": round(32 / (ms / 1e3), 1), "unit": "frames/s",
                                 "GBps": round(32 * w * h * 3 / ms / 1e6, 2),
                                 "what": "32 P6 frames 1352x1014 (page cache) -> pinned u8 array, all host threads"}
    rng = np.random.default_rng(1)
    pos, col = rng.uniform(-3, 3, (100_000, 3)), rng.uniform(0, 1, (100_000, 3))
    ctx.init_scene(pos[:1000], col[:1000])
    ms, _ = wall(lambda: ctx.init_scene(pos, col, A.InitConfig(sh_degree=3)))
    out["init_scene"] = {"ms": round(ms, 2), "points": 100_000, "pairs_per_s": round(1e5 * 1e5 / (ms / 1e3), 1),
                         "what": "FP64 brute-force 3-NN over 100k points + field init (data_io.cpp:189-238)"}
    return out


def cpu_baseline(scene, cam, t, gt) -> dict:
    """The oracle (FP64 CPU restatement of the reference) on one full c2 view:
    tiled taped forward on all cores, L1+SSIM, backward (single-threaded, as
    the reference), Adam.  Bounded sample: one iteration (~10-30 s)."""
    import oracle as O

    s = scene.copy()
    st = O.AdamState(s)
    cores = O.hardware_threads()
    t0 = time.perf_counter()
    O.train_step(s, st, [cam], [t], [gt], (0.2, 0.2, 0.2), num_threads=1, tile_threads=cores)
    dt = time.perf_counter() - t0
    return {"value": round(1.0 / dt, 5), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"one full {cam.width}x{cam.height} training iteration of the c2 scene "
                      f"({dt:.2f} s): tiled forward w/ tape on {cores} threads, L1+SSIM, backward 1 thread, Adam",
            "literal_forward_train": literal_forward_train(scene, cam, t)}


def literal_forward_train(scene, cam, t) -> dict:
    """The reference's own forward_train is UNTILED (backward.cpp:142-175:
    every projected splat tested at every pixel).  Timed on one thread, as the
    reference, at 1/256 of c2's pixels x Gaussians (N/4 Gaussians, W/8 x H/8
    pixels) and extrapolated x256 (the cost is linear in both)."""
    import oracle as O
    from paper_2505_13215_b200.scene import Camera

    sub = scene.subset(scene.n4 // 4, scene.n3 // 4) if hasattr(scene, "subset") else None
    if sub is None:
        return {"note": "scene subset unavailable"}
    small = Camera(fx=cam.fx / 8, fy=cam.fy / 8, cx=cam.cx / 8, cy=cam.cy / 8, rot=cam.rot, trans=cam.trans,
                   width=cam.width // 8, height=cam.height // 8, near=cam.near, far=cam.far)
    try:  # the reference's own forward_train (oracle/_ref, compiled from its sources) when built
        from oracle import ref as R

        use_ref = R.available()
    except Exception:
        use_ref = False
    t0 = time.perf_counter()
    if use_ref:
        R.forward_backward(sub, small, t, (0.2, 0.2, 0.2), None)
    else:
        O.forward_train(sub, small, t, (0.2, 0.2, 0.2), untiled=True)
    dt = time.perf_counter() - t0
    return {"seconds_at_1_256": round(dt, 3), "extrapolated_s_per_c2_view": round(256 * dt, 1),
            "views_per_s": round(1.0 / (256 * dt), 6), "cores": 1,
            "kind": "reference" if use_ref else "port",
            "sample": f"{sub.n4 + sub.n3} Gaussians, {small.width}x{small.height}, untiled taped forward only "
                      f"({'hgs::forward_train of the reference compiled from its sources' if use_ref else 'oracle restatement'})"}


# ------------------------------------------------------------------ reference arm
def run_reference(args) -> None:
    """The reference's CPU path for the same workload and config as the GPU
    arm (c2, full 1352x1014 views; at N GPUs the same N views per
    iteration): the FP64 oracle port of proj/src (pinned bit for bit against
    the reference built from its sources, oracle/_ref), forward tiled with
    its tape on all host threads (RasterOpts::num_threads,
    raster.cpp:150-163), L1 + D-SSIM, backward on one thread as the
    reference, Adam.  The reference's own training forward is the untiled
    forward_train (backward.cpp:142-175), ~45 min per c2 view on one core:
    it is timed on a 1/256 sample in the GPU arm's
    cpu_baseline.literal_forward_train; this arm uses the (faster,
    conservative) tiled port.  Steps are bounded to ceil(steps / N)
    iterations so the run stays within minutes.  Under torchrun only rank 0
    runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    from paper_2505_13215_b200.train import quantize_8bit

    scene, target, cams, times, desc = workload(args.config)
    cores = O.hardware_threads()
    gts = {}

    def gt(v):
        if v not in gts:
            gts[v] = quantize_8bit(O.rasterize(target, cams[v], times[v], (0.2, 0.2, 0.2), num_threads=cores)["rgb"])
        return gts[v]

    s = scene.copy()
    st = O.AdamState(s)

    world = max(1, args.gpus)
    steps = max(1, -(-args.steps // world))  # bounded sample: ceil(steps / N) iterations of N views

    def views(i):
        return [(i * world + r) % len(cams) for r in range(world)]

    def step(i):
        vs = views(i)
        O.train_step(s, st, [cams[v] for v in vs], [times[v] for v in vs], [gt(v) for v in vs], (0.2, 0.2, 0.2),
                     num_threads=1, tile_threads=cores)

    for i in range(args.warmup + steps):
        for v in views(i):
            gt(v)  # ground truth rendered outside the timed steps
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = steps * world / dt
    sample = (f"{steps} training iteration(s) of {world} full {cams[0].width}x{cams[0].height} c2 view(s), "
              f"forward tiled on {cores} threads, backward 1 thread; FP64 oracle port of the reference")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / steps * 1e3, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           # the GPU arm's config, key for key (same workload, same views per iteration)
           "config": dict(desc, parallelism=f"view-parallel dp{world}", views_per_iteration=world),
           "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
           "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def self_launch(args) -> int | None:
    """`bench.py --gpus N` outside torchrun: start N ranks with
    torch.distributed.run on 127.0.0.1 and return their exit code; under
    torchrun, insist that WORLD_SIZE == --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return None
    if args.gpus <= 1:
        return None
    import socket

    import torch

    if torch.cuda.device_count() < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} CUDA devices")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c1/c5 render and c4 training lines")
    ap.add_argument("--view-parallel", action="store_true",
                    help="use the N-GPU code path (NCCL exchange) even on one GPU (a one-rank communicator)")
    ap.add_argument("--sharded", action="store_true",
                    help="view-parallel path with the sharded optimizer exchange (reduce-scatter -> Adam on the "
                         "rank's shard -> all-gather) instead of the gradient all-reduce")
    ap.add_argument("--no-phase-profile", action="store_true",
                    help="no per-phase CUDA events in the timed region (roofline.kernels then empty)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    run_ours(args)


if __name__ == "__main__":
    main()
