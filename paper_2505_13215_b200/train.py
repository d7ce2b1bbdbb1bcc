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


def linear_to_srgb8(v: np.ndarray) -> np.ndarray:
    """image.cpp:15-18"""
    v = np.clip(v, 0.0, 1.0)
    return np.rint(np.power(v, 1.0 / 2.2) * 255.0).astype(np.uint8)


def srgb8_to_linear(v: np.ndarray) -> np.ndarray:
    """image.cpp:20-22"""
    return np.power(v.astype(np.float64) / 255.0, 2.2)


def quantize_8bit(img: np.ndarray) -> np.ndarray:
    """image.cpp:77-82: the PPM save/load round trip, pixel for pixel."""
    return srgb8_to_linear(linear_to_srgb8(img))


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


class DeviceTrainer:
    """Single-GPU (or one-rank) trainer around a Context.

    ``target`` (a HybridScene) renders the ground truth on the device through
    the parity-validated forward path; alternatively pass ``gt_images``.
    """

    def __init__(self, ctx: Context, scene: HybridScene, cameras: list[Camera], times: list[float],
                 target: HybridScene | None = None, gt_images: list[np.ndarray] | None = None,
                 bg=(0.0, 0.0, 0.0), ssim_lambda: float = 0.2, lrs: LearningRates | None = None,
                 iterations: int = 2000, weight_cutoff: float = 0.05, quantize_gt: bool = True):
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
        if gt_images is None:
            if target is None:
                raise ValueError("DeviceTrainer: need target or gt_images")
            ctx.upload(target)
            gt_images = []
            for cam, t in zip(self.cameras, self.times):
                img = ctx.render(cam, t, self.bg, weight_cutoff=weight_cutoff)["rgb"].astype(np.float64)
                gt_images.append(quantize_8bit(img) if quantize_gt else img)
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

    def adam(self) -> int:
        return self.ctx.adam_step(self.lrs, self.decay())


class ViewParallelTrainer(DeviceTrainer):
    """One rank of the view-parallel trainer (torch.distributed, NCCL on GPUs,
    gloo on CPU for the host-logic tests)."""

    def __init__(self, *args, group=None, **kw):
        super().__init__(*args, **kw)
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def grads_tensor(self):
        ptr, n = self.ctx.grads_device()
        return self.torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{self.ctx.device}")

    def step(self, batch: list[int], batch_total: int | None = None, apply_adam: bool = True) -> float:
        mine = shard_batch(batch, self.rank, self.world)
        self.iter += 1
        loss = DeviceTrainer.step(self, mine, batch_total=len(batch), apply_adam=False) * max(1, len(mine))
        g = self.grads_tensor()
        self.dist.all_reduce(g, group=self.group)          # sum of dense grads + stat deltas
        lt = self.torch.tensor([loss], dtype=self.torch.float64, device=g.device)
        self.dist.all_reduce(lt, group=self.group)
        self.ctx.adam_step(self.lrs, self.decay())
        return float(lt.item()) / len(batch)


def shard_batch(batch: list[int], rank: int, world: int) -> list[int]:
    """Rank r takes batch items {b : b mod world == r}."""
    return [v for i, v in enumerate(batch) if i % world == rank]


def sample_batches(n_samples: int, batch_size: int, iterations: int, seed: int) -> list[list[int]]:
    """Deterministic batch schedule shared by all ranks (train.cpp:387-404
    samples (camera, frame) pairs uniformly; every rank draws the same list)."""
    rng = np.random.default_rng(seed)
    return [list(rng.integers(0, n_samples, batch_size)) for _ in range(iterations)]
