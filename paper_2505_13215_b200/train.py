"""Device-resident training driver over the C ABI (train.cpp:382-494 loop).

The per-iteration work -- render every batch view, L1+D-SSIM loss, backward
scaled by 1/B, Adam -- is one ``hgs_train_step`` call; the scene, its Adam
state and the ground-truth frames never leave HBM.  Ground-truth frames are
device tensors (torch is used here only as the device-memory allocator).

View-parallel multi-GPU: every rank holds a full replica, the
batch is sampled identically on every rank and rank r renders batch items
{b : b mod n == r}; the packed gradient buffer (parameter gradients plus this
step's densification-statistic deltas, one contiguous FP32 payload) is summed
with one NCCL all-reduce, after which every rank applies the same Adam step,
so replicas stay bit-identical without a broadcast.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _capi
from .api import Context, LearningRates
from .scene import Camera, HybridScene


# image.cpp:20-22 srgb8_to_linear for every code, with the C library's pow
SRGB8_LUT = np.array([math.pow(v / 255.0, 2.2) for v in range(256)])


def linear_to_srgb8(v: np.ndarray) -> np.ndarray:
    """image.cpp:15-18 (std::lround: halves away from zero)"""
    v = np.clip(v, 0.0, 1.0)
    return np.floor(np.power(v, 1.0 / 2.2) * 255.0 + 0.5).astype(np.uint8)


def srgb8_to_linear(v: np.ndarray) -> np.ndarray:
    """image.cpp:20-22"""
    return SRGB8_LUT[np.asarray(v, dtype=np.uint8)]


def quantize_8bit(img: np.ndarray) -> np.ndarray:
    """image.cpp:77-82: the PPM save/load round trip, pixel for pixel."""
    return srgb8_to_linear(linear_to_srgb8(img))


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def render_gt_u8_device(ctx: Context, target: HybridScene, cameras: list, times: list, bg=(0.0, 0.0, 0.0),
                        weight_cutoff: float = 0.05) -> list:
    """Ground-truth frames as the reference's dataset holds them (8-bit sRGB,
    image.cpp:15-18), rendered and encoded on the device: one device u8 HWC
    tensor per (camera, time).  For dataset-sized frame counts (configs[2]:
    18 cameras x 300 frames) where the host round trip per frame would
    dominate.  Uploads ``target`` (the caller uploads its own scene after)."""
    import torch

    ctx.upload(target)
    out = []
    for cam, t in zip(cameras, times):
        ctx.render_device(cam, t, bg, weight_cutoff=weight_cutoff)
        n = cam.height * cam.width * 3
        img = torch.as_tensor(_CudaArray(ctx.last_image_device_ptr(), n), device=f"cuda:{ctx.device}")
        v = img.double().clamp(0.0, 1.0).pow(1.0 / 2.2).mul(255.0).add(0.5).floor()
        out.append(v.to(torch.uint8).view(cam.height, cam.width, 3).clone())
        torch.cuda.synchronize(ctx.device)  # the next render reuses the context's image buffer
    return out


class DeviceTrainer:
    """Single-GPU (or one-rank) trainer around a Context.

    ``target`` (a HybridScene) renders the ground truth on the device through
    the parity-validated forward path; alternatively pass ``gt_images``.
    """

    def __init__(self, ctx: Context, scene: HybridScene, cameras: list[Camera], times: list[float],
                 target: HybridScene | None = None, gt_images: list[np.ndarray] | None = None,
                 bg=(0.0, 0.0, 0.0), ssim_lambda: float = 0.2, lrs: LearningRates | None = None,
                 iterations: int = 2000, weight_cutoff: float = 0.05, quantize_gt: bool = True,
                 gt_format: str = "f32", gt_device: list | None = None):
        """gt_format: "f32" -- linear float frames on the device; "u8" -- the
        8-bit sRGB codes (4x smaller), decoded inside the loss (HGS_U8).
        gt_device: ready device frames in that format (torch tensors, HWC),
        e.g. from render_gt_u8_device; then neither target nor gt_images."""
        import torch

        self.torch = torch
        self.ctx = ctx
        self.cameras = list(cameras)
        self.times = list(times)
        self.bg = tuple(float(b) for b in bg)
        self.ssim_lambda = ssim_lambda
        self.lrs = lrs or LearningRates()
        self.iterations = iterations
        self.weight_cutoff = weight_cutoff
        self.iter = 0
        dev = torch.device("cuda", ctx.device)
        if gt_device is not None:
            gt_images = []
        if gt_images is None:
            if target is None:
                raise ValueError("DeviceTrainer: need target or gt_images")
            ctx.upload(target)
            gt_images = []
            for cam, t in zip(self.cameras, self.times):
                img = ctx.render(cam, t, self.bg, weight_cutoff=weight_cutoff)["rgb"].astype(np.float64)
                gt_images.append(quantize_8bit(img) if quantize_gt else img)
        if gt_format not in ("f32", "u8"):
            raise ValueError("gt_format: 'f32' or 'u8'")
        self.gt_format = gt_format
        if gt_device is not None:
            self.gt = list(gt_device)
        elif gt_format == "u8":
            self.gt = [torch.as_tensor(np.ascontiguousarray(linear_to_srgb8(g)), device=dev) for g in gt_images]
        else:
            self.gt = [torch.as_tensor(np.ascontiguousarray(g, dtype=np.float32), device=dev) for g in gt_images]
        ctx.upload(scene)
        self._cams = (_capi.Camera_ * max(1, len(self.cameras)))()
        for i, c in enumerate(self.cameras):
            self._cams[i] = _capi.camera_struct(c)

    def _opts(self, decay: float) -> _capi.TrainOpts:
        o = _capi.TrainOpts()
        o.ssim_lambda, o.weight_cutoff, o.mean_lr_scale = self.ssim_lambda, self.weight_cutoff, decay
        o.lrs = self.lrs.struct()
        for i in range(3):
            o.bg[i] = self.bg[i]
        return o

    def decay(self) -> float:
        """train.cpp:449: mean_final_ratio ** (iter / iterations)."""
        return math.pow(self.lrs.mean_final_ratio, self.iter / max(1, self.iterations))

    def step(self, views: list[int], batch_total: int | None = None, apply_adam: bool = True) -> float:
        """One iteration over ``views`` (indices into cameras); returns the mean loss."""
        if self.gt_format == "u8":
            self.step_async(views, batch_total, apply_adam)
            return self.collect()
        if apply_adam:
            self.iter += 1
        n = len(views)
        cams = (_capi.Camera_ * max(1, n))(*[self._cams[v] for v in views])
        times = (C.c_double * max(1, n))(*[self.times[v] for v in views])
        gts = (_capi._fp * max(1, n))(*[C.cast(C.c_void_p(self.gt[v].data_ptr()), _capi._fp) for v in views])
        loss = C.c_double()
        bt = batch_total or n
        self.ctx._check(self.ctx._lib.hgs_train_step(self.ctx.handle, n, cams, times, gts, bt,
                                                     C.byref(self._opts(self.decay())), 1 if apply_adam else 0,
                                                     C.byref(loss)))
        return loss.value / max(1, n)

    def step_async(self, views: list[int], batch_total: int | None = None, apply_adam: bool = True,
                   gt_host: list | None = None) -> None:
        """Enqueue one iteration (hgs_train_step_async) without waiting for it;
        ``collect()`` returns the mean losses in order.  ``gt_host``: pinned
        host float32 frames per view instead of the device-resident ones."""
        if apply_adam:
            self.iter += 1
        n = len(views)
        cams = (_capi.Camera_ * max(1, n))(*[self._cams[v] for v in views])
        times = (C.c_double * max(1, n))(*[self.times[v] for v in views])
        src = gt_host if gt_host is not None else [self.gt[v] for v in views]
        gts = (C.c_void_p * max(1, n))(*[C.c_void_p(t.data_ptr()) for t in src])
        dtype = _capi.HGS_U8 if src and src[0].dtype == self.torch.uint8 else _capi.HGS_F32
        self.ctx._check(self.ctx._lib.hgs_train_step_async(self.ctx.handle, n, cams, times, gts, dtype,
                                                           0 if gt_host is not None else 1, batch_total or n,
                                                           C.byref(self._opts(self.decay())),
                                                           1 if apply_adam else 0))
        self._pending_n = getattr(self, "_pending_n", [])
        self._pending_n.append(n)

    def collect(self) -> float:
        """Mean loss of the oldest enqueued iteration (raises NumericAbort)."""
        loss = C.c_double()
        n = self._pending_n.pop(0)
        rc = self.ctx._lib.hgs_train_collect(self.ctx.handle, C.byref(loss))
        if rc != 0:
            self._pending_n.clear()
        self.ctx._check(rc)
        return loss.value / max(1, n)

    def adam(self) -> int:
        return self.ctx.adam_step(self.lrs, self.decay())


class ViewParallelTrainer(DeviceTrainer):
    """One rank of the view-parallel trainer (torch.distributed, NCCL on GPUs,
    gloo on CPU for the host-logic tests)."""

    def __init__(self, *args, group=None, exchange: str = "torch", verify_every: int = 0, sharded: bool = False,
                 **kw):
        """exchange: "torch" -- torch.distributed all-reduce of the packed
        payload; "capi" -- the library's own NCCL communicator
        (hgs_allreduce_grads).  verify_every > 0: every that many steps the
        ranks compare parameter checksums and, on a mismatch, reload rank 0's
        state (SURVEY.md 8e replica consistency)."""
        super().__init__(*args, **kw)
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if exchange not in ("torch", "capi"):
            raise ValueError("exchange: 'torch' or 'capi'")
        self.exchange = exchange
        self.verify_every = verify_every
        self.repairs = 0
        if exchange == "capi" and getattr(self.ctx, "_comm_world", None) != self.world:
            # one communicator per context: a second trainer on the same
            # context (another scene) reuses it
            uid = [Context.comm_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(uid, src=0, group=group)
            self.ctx.comm_init(self.world, self.rank, uid[0])
        # sharded=True (exchange "capi", pipelined steps): reduce-scatter ->
        # Adam on this rank's shard -> all-gather; gather_state() before
        # densification / sweeps / checkpoints with optimizer state
        if sharded and exchange != "capi":
            raise ValueError("sharded exchange needs exchange='capi'")
        self.sharded = sharded
        if exchange == "capi":
            self.ctx.set_sharded(sharded)

    def grads_tensor(self):
        ptr, n = self.ctx.grads_device()
        return self.torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{self.ctx.device}")

    def packed_grads_tensor(self):
        """The packed payload (valid gradient rows + stat deltas, no capacity padding)."""
        ptr, n = self.ctx.grads_packed()
        return self.torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{self.ctx.device}")

    def step(self, batch: list[int], batch_total: int | None = None, apply_adam: bool = True) -> float:
        mine = shard_batch(batch, self.rank, self.world)
        self.iter += 1
        loss = DeviceTrainer.step(self, mine, batch_total=len(batch), apply_adam=False) * max(1, len(mine))
        # the batch loss first: every rank takes the same NumericAbort decision
        # (train.cpp:445-447) before any collective on the gradients
        try:
            total = reduce_batch_loss(self.dist, self.group, loss, f"cuda:{self.ctx.device}")
        except _capi.NumericAbort:
            self.ctx.zero_grads()
            raise
        if self.exchange == "capi":
            self.ctx.allreduce_grads()                     # pack -> ncclAllReduce -> unpack, one stream
        else:
            g = self.packed_grads_tensor()
            self.dist.all_reduce(g, group=self.group)      # sum of dense grads + stat deltas
            self.ctx.grads_unpack()
        self.ctx.adam_step(self.lrs, self.decay())
        if self.verify_every and self.iter % self.verify_every == 0:
            self.verify_replicas()
        return total / len(batch)

    def step_async(self, batch: list[int], batch_total: int | None = None, apply_adam: bool = True,
                   gt_host: list | None = None) -> None:
        """Pipelined view-parallel iteration (exchange="capi"): this rank's
        views, then hgs_train_exchange_async (all-reduced loss gate + packed
        gradients + gated Adam) -- no host synchronisation; collect() returns
        this rank's mean view loss later and raises NumericAbort on every rank
        for the same iteration."""
        if self.exchange != "capi":
            raise ValueError("step_async needs exchange='capi'")
        mine = shard_batch(batch, self.rank, self.world)
        self.iter += 1
        DeviceTrainer.step_async(self, mine, batch_total=len(batch), apply_adam=False, gt_host=gt_host)
        self.ctx._check(self.ctx._lib.hgs_train_exchange_async(self.ctx.handle, C.byref(self._opts(self.decay()))))

    def gather_state(self) -> None:
        """Whole Adam moments on every rank (call on every rank after sharded
        steps, before densify / sweep_convert / save_checkpoint)."""
        while self.ctx._lib.hgs_train_pending(self.ctx.handle):
            self.collect()
        self.ctx.gather_state()

    def verify_replicas(self) -> bool:
        """True when every rank's parameters hash equal; otherwise rank 0's
        scene, optimizer state and statistics are shipped to every rank
        (as a checkpoint image) and False is returned."""
        ok = replicas_agree(self.dist, self.group, self.ctx.param_checksum())
        if not ok:
            repair_from_root(self.dist, self.group, self.rank, self.ctx)
            self.repairs += 1
        return ok


def replicas_agree(dist, group, checksum: int) -> bool:
    """All ranks hold the same 64-bit parameter checksum."""
    allv = [None] * dist.get_world_size(group)
    dist.all_gather_object(allv, int(checksum), group=group)
    return all(v == allv[0] for v in allv)


def repair_from_root(dist, group, rank: int, ctx, root: int = 0) -> None:
    """Every rank takes the root's device state (parameters, Adam moments,
    statistics, step) through the checkpoint encoder / decoder."""
    import os
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, f"replica{rank}.hgsc")
        blob = [None]
        if rank == root:
            ctx.save_checkpoint(path)
            with open(path, "rb") as f:
                blob[0] = f.read()
        dist.broadcast_object_list(blob, src=root, group=group)
        if rank != root:
            with open(path, "wb") as f:
                f.write(blob[0])
            ctx.load_checkpoint(path)


def reduce_batch_loss(dist, group, local_loss: float, device: str = "cpu") -> float:
    """Sum of the ranks' view losses; every rank raises NumericAbort together
    when it is non-finite (train.cpp:445-447), before any gradient collective."""
    import torch

    lt = torch.tensor([local_loss], dtype=torch.float64, device=device)
    dist.all_reduce(lt, group=group)
    total = float(lt.item())
    if not math.isfinite(total):
        raise _capi.NumericAbort("train: non-finite loss")
    return total


def shard_batch(batch: list[int], rank: int, world: int) -> list[int]:
    """Rank r takes batch items {b : b mod world == r}."""
    return [v for i, v in enumerate(batch) if i % world == rank]


def sample_batches(n_samples: int, batch_size: int, iterations: int, seed: int) -> list[list[int]]:
    """Deterministic batch schedule shared by all ranks (train.cpp:387-404
    samples (camera, frame) pairs uniformly; every rank draws the same list)."""
    from .api import Rng

    r = Rng(seed)
    return [r.batch(n_samples, batch_size) for _ in range(iterations)]


# --------------------------------------------------------------------------
# train_scene: the reference's training loop (train.cpp:382-494), device
# resident.  Same configuration, same batch schedule (std::mt19937_64 +
# uniform_int_distribution restated bit-exactly in rng.py), same cadence of
# Adam / decay / densify (device) / sweep / probe.

from dataclasses import dataclass, field  # noqa: E402



@dataclass
class TrainConfig:  # train.hpp:23-49
    iterations: int = 2000
    batch_size: int = 2
    warmup_iters: int = 500
    densify_interval: int = 100
    densify_stop_iter: int = 1500
    grad_threshold: float = 0.02
    opacity_prune_eps: float = 0.005
    tau: float = 0.5
    conversion_enabled: bool = True
    ssim_lambda: float = 0.2
    lrs: LearningRates = field(default_factory=LearningRates)
    opacity_reset_enabled: bool = False
    opacity_reset_interval: int = 600
    seed: int = 0
    sh_degree: int = 1
    weight_cutoff: float = 0.05
    max_gaussians: int = 20000
    clone_size_frac: float = 0.01
    split_factor: float = 1.6
    num_threads: int = 1
    probe_interval: int = 100
    init_temporal_scale: float = 0.1
    init_opacity: float = 0.1

    _FILE_KEYS = ("iterations", "batch_size", "warmup_iters", "densify_interval", "densify_stop_iter",
                  "grad_threshold", "opacity_prune_eps", "tau", "conversion_enabled", "ssim_lambda",
                  "opacity_reset_enabled", "opacity_reset_interval", "seed", "sh_degree", "weight_cutoff",
                  "max_gaussians", "num_threads", "probe_interval", "init_temporal_scale", "init_opacity")
    _LR_KEYS = (("lr_mean", "mean"), ("lr_mean_final_ratio", "mean_final_ratio"), ("lr_mean_t", "mean_t"),
                ("lr_quat", "quat"), ("lr_scales", "scales"), ("lr_opacity", "opacity"), ("lr_sh", "sh"))

    @classmethod
    def from_file(cls, path: str) -> "TrainConfig":
        """TrainConfig::from_file (train.cpp:87-120): `key = value` lines
        (config.cpp KeyValueFile rules), unknown keys are a FormatError,
        then validate()."""
        from .dataset import KeyValueFile

        kv = KeyValueFile(path)
        cfg = cls()
        for k in cls._FILE_KEYS:
            cur = getattr(cfg, k)
            if isinstance(cur, bool):
                setattr(cfg, k, kv.get_bool(k, cur))
            elif k == "seed":
                setattr(cfg, k, kv.get_uint(k, cur))
            elif isinstance(cur, int):
                setattr(cfg, k, kv.get_int(k, cur))
            else:
                setattr(cfg, k, kv.get_float(k, cur))
        for k, attr in cls._LR_KEYS:
            setattr(cfg.lrs, attr, kv.get_float(k, getattr(cfg.lrs, attr)))
        kv.finish()
        cfg.validate()
        return cfg

    def validate(self) -> None:  # train.cpp:76-85 (TrainConfig::validate)
        if self.warmup_iters > self.iterations and self.iterations > 0:
            raise ValueError("TrainConfig: warmup_iters must be <= iterations")
        if self.densify_interval < 1:
            raise ValueError("TrainConfig: densify_interval must be >= 1")
        if self.ssim_lambda < 0.0 or self.ssim_lambda > 1.0:
            raise ValueError("TrainConfig: ssim_lambda must be in [0,1]")
        if self.batch_size < 1:
            raise ValueError("TrainConfig: batch_size must be >= 1")
        if not self.tau > 0.0:
            raise ValueError("TrainConfig: tau must be positive")

    def densifies(self) -> bool:
        """Would train.cpp:456-458 call densify_and_prune at some iteration?"""
        first = max(self.warmup_iters, 1)
        first += (-first) % self.densify_interval
        return first <= min(self.iterations, self.densify_stop_iter)


@dataclass
class Frame:  # data_io.hpp Frame: one image of one camera at one time
    time: float
    image: np.ndarray  # (H, W, 3): float linear RGB, or uint8 sRGB codes (decoded on the device)


@dataclass
class MultiViewDataset:  # data_io.hpp:28-41 MultiViewDataset
    cameras: list
    frames: list  # frames[camera][frame] -> Frame
    background: tuple = (0.0, 0.0, 0.0)
    duration_seconds: float = 1.0
    camera_ids: list = field(default_factory=list)
    init_points: object = None  # dataset.InitPoints (root/points.txt)

    def total_frames(self) -> int:
        return sum(len(f) for f in self.frames)


@dataclass
class TrainLogRow:  # train.hpp:51-58
    iter: int = 0
    loss: float = 0.0
    probe_psnr: float = -1.0
    n_static: int = 0
    n_dynamic: int = 0
    conversions: int = 0
    wall_seconds: float = 0.0


def write_train_log_csv(rows: list, path: str) -> None:
    """TrainLog::write_csv (train.cpp:122-129)."""
    with open(path, "w") as f:
        f.write("iter,loss,probe_psnr,n_static,n_dynamic,conversions,wall_seconds\n")
        for r in rows:
            f.write(f"{r.iter},{r.loss:.6g},{r.probe_psnr:.6g},{r.n_static},{r.n_dynamic},{r.conversions},"
                    f"{r.wall_seconds:.6g}\n")


@dataclass
class TrainResult:  # train.hpp:80-84 (state = Adam moments m, v and the step)
    scene: HybridScene
    log: list
    state: tuple


from .api import psnr, ssim  # noqa: E402,F401  (device metrics, metrics.cpp:91-101)


@dataclass
class MetricReport:  # metrics.hpp:21-29
    frame_psnr: list = field(default_factory=list)
    frame_ssim: list = field(default_factory=list)
    mean_psnr: float = 0.0
    mean_ssim: float = 0.0
    frames: int = 0

    def add(self, p: float, s: float) -> None:  # metrics.cpp:109-120
        self.frame_psnr.append(p)
        self.frame_ssim.append(s)
        self.frames = len(self.frame_psnr)
        sp = ss = 0.0
        for i in range(self.frames):
            sp += self.frame_psnr[i]
            ss += self.frame_ssim[i]
        self.mean_psnr = sp / self.frames
        self.mean_ssim = ss / self.frames


def evaluate_views(scene: HybridScene | None, dataset: MultiViewDataset, weight_cutoff: float = 0.05,
                   ctx: Context | None = None) -> MetricReport:
    """eval.cpp:12-23 on the device: renders every (camera, frame) of the
    dataset and scores it (PSNR + SSIM) without downloading the image.
    ``scene`` is uploaded into ``ctx`` first unless None (score the resident
    scene).  Frames may be float (linear) or uint8 (sRGB) arrays."""
    ctx = ctx or Context(0)
    if scene is not None:
        ctx.upload(scene)
    report = MetricReport()
    for ci, cam in enumerate(dataset.cameras):
        for fr in dataset.frames[ci]:
            ctx.render_device(cam, fr.time, dataset.background, weight_cutoff=weight_cutoff)
            report.add(*ctx.image_metrics(fr.image))
    return report


def train_scene(scene: HybridScene, dataset: MultiViewDataset, cfg: TrainConfig, ctx: Context | None = None,
                state: tuple | None = None, on_row=None) -> TrainResult:
    """train.cpp:382-494 on the device: ``state`` = (m, v, step) to continue
    from (checkpoints), ``on_row`` is called with each TrainLogRow."""
    import time as _time

    import torch

    if not dataset.cameras or dataset.total_frames() == 0:  # train.cpp:367-368
        raise ValueError("train: dataset is empty")
    cfg.validate()
    from .api import default_context

    ctx = ctx or default_context()
    scene = scene.copy()
    scene.tau = cfg.tau
    ctx.upload(scene)
    if state is not None:
        ctx.set_adam_state(*state)
    dev = torch.device("cuda", ctx.device)
    samples = [(c, f) for c in range(len(dataset.frames)) for f in range(len(dataset.frames[c]))]
    # 8-bit sRGB frames (dataset.load_dataset) stay 8-bit on the device and
    # are decoded inside the loss (HGS_U8); float frames are linear RGB
    u8 = dataset.frames[0][0].image.dtype == np.uint8
    gts = {(c, f): torch.as_tensor(np.ascontiguousarray(dataset.frames[c][f].image,
                                                        dtype=np.uint8 if u8 else np.float32), device=dev)
           for c, f in samples}
    cams = [_capi.camera_struct(c) for c in dataset.cameras]
    from .api import Rng

    rng = Rng(cfg.seed)  # libstdc++ mt19937_64 stream shared by batches and densification (train.cpp:387)
    probe = (0, len(dataset.frames[0]) // 2)
    o = _capi.TrainOpts()
    o.ssim_lambda, o.weight_cutoff = cfg.ssim_lambda, cfg.weight_cutoff
    o.lrs = cfg.lrs.struct()
    for i in range(3):
        o.bg[i] = float(dataset.background[i])
    B = cfg.batch_size
    log = []
    t0 = _time.perf_counter()
    for it in range(1, cfg.iterations + 1):
        batch = [samples[i] for i in rng.batch(len(samples), B)]  # train.cpp:403-404
        o.mean_lr_scale = math.pow(cfg.lrs.mean_final_ratio, it / cfg.iterations)  # train.cpp:449
        karr = (_capi.Camera_ * B)(*[cams[c] for c, _ in batch])
        tarr = (C.c_double * B)(*[dataset.frames[c][f].time for c, f in batch])
        loss = C.c_double()
        # renders, losses, backward scaled by 1/B, densify statistics, NumericAbort, Adam
        if u8:
            garr = (C.c_void_p * B)(*[C.c_void_p(gts[b].data_ptr()) for b in batch])
            ctx._check(ctx._lib.hgs_train_step_async(ctx.handle, B, karr, tarr, garr, _capi.HGS_U8, 1, B, C.byref(o), 1))
            ctx._check(ctx._lib.hgs_train_collect(ctx.handle, C.byref(loss)))
        else:
            garr = (_capi._fp * B)(*[C.cast(C.c_void_p(gts[b].data_ptr()), _capi._fp) for b in batch])
            ctx._check(ctx._lib.hgs_train_step(ctx.handle, B, karr, tarr, garr, B, C.byref(o), 1, C.byref(loss)))
        row = TrainLogRow(iter=it, loss=loss.value / B)
        if it >= cfg.warmup_iters and it % cfg.densify_interval == 0:
            if it <= cfg.densify_stop_iter:  # train.cpp:457-465, on the device
                ctx.densify_and_prune(rng, cfg.grad_threshold, cfg.opacity_prune_eps, cfg.clone_size_frac,
                                      cfg.split_factor, cfg.max_gaussians)
                if cfg.opacity_reset_enabled and cfg.opacity_reset_interval > 0 and \
                        it % cfg.opacity_reset_interval == 0:
                    ctx.opacity_reset()
            if cfg.conversion_enabled:
                moved, _ = ctx.sweep_convert()  # train.cpp:466-472 (Adam rows remapped on the device)
                row.conversions = len(moved)
        if cfg.probe_interval > 0 and (it % cfg.probe_interval == 0 or it == cfg.iterations):
            pf = dataset.frames[probe[0]][probe[1]]
            ctx.render_device(dataset.cameras[probe[0]], pf.time, dataset.background,
                              weight_cutoff=cfg.weight_cutoff)
            row.probe_psnr = ctx.image_metrics(pf.image, want_ssim=False)[0]
        row.n_dynamic, row.n_static = ctx.counts()
        row.wall_seconds = _time.perf_counter() - t0
        log.append(row)
        if on_row:
            on_row(row)
    return TrainResult(scene=ctx.download(), log=log, state=ctx.adam_state())


def train(dataset: MultiViewDataset, cfg: TrainConfig, ctx: Context | None = None, on_row=None) -> TrainResult:
    """hgs::train (train.cpp:366-380): init_scene from the dataset's points
    (the GPU kNN, api.Context.init_scene), then train_scene."""
    if not dataset.cameras or dataset.total_frames() == 0:
        raise ValueError("train: dataset is empty")
    from .api import InitConfig, default_context

    ctx = ctx or default_context()
    pts = dataset.init_points
    if pts is None or len(pts) < 4:
        raise ValueError("init_scene: need at least 4 points")
    ctx.init_scene(pts.positions, pts.rgb, InitConfig(sh_degree=cfg.sh_degree, tau=cfg.tau,
                                                      duration_seconds=dataset.duration_seconds,
                                                      init_temporal_scale=cfg.init_temporal_scale,
                                                      init_opacity=cfg.init_opacity))
    return train_scene(ctx.download(), dataset, cfg, ctx=ctx, on_row=on_row)


def train_directory(data_dir: str, held_out: int = -1, config: TrainConfig | None = None,
                    ctx: Context | None = None):
    """hybridgs.train (bindings.cpp:221-235): load the dataset directory
    (8-bit frames), train, and score the held-out camera -> (scene,
    held_out_psnr); held_out_psnr is -1 without a held-out camera."""
    from . import dataset as D
    from .api import default_context

    cfg = config or TrainConfig()
    split, held = D.load_dataset(data_dir, held_out)
    ctx = ctx or default_context()
    result = train(split, cfg, ctx=ctx)
    held_psnr = -1.0
    if held.cameras:
        held_psnr = evaluate_views(None, held, cfg.weight_cutoff, ctx=ctx).mean_psnr
    return result.scene, held_psnr
