"""Python mirror of the reference's render/train surface over the C ABI.

The reference exposes its C++ library to Python as ``hybridgs._core``
(python/bindings.cpp:35-236): ``rasterize(scene, camera, t, background,
num_threads, weight_cutoff)`` etc.  The same names and argument meanings are
provided here, backed by the sm_100a kernels in libhgs_gpu.so; scenes are the
SoA :class:`~paper_2505_13215_b200.scene.HybridScene`.  Errors map to the
reference's exception types (``ValueError`` for std::invalid_argument,
``DegenerateTemporalError`` ...).

:class:`Context` is the device-resident API (one per GPU): the scene, Adam
state and gradients stay in HBM across calls, which is how the training loop
uses it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import (HGS_F32, HGS_F64, HGS_U8, CudaError, DegenerateRotationError, DegenerateTemporalError,  # noqa: F401
                    FormatError, HgsError, IntegrityError, NumericAbort, StateError, UnsupportedVersionError, check,
                    check_io, ptr)
from .scene import Camera, HybridScene, sh_coeff_count

DEFAULT_WEIGHT_CUTOFF = 0.05  # raster.hpp:19


@dataclass
class LearningRates:  # train.hpp:13-21
    mean: float = 1.6e-4
    mean_final_ratio: float = 0.01
    mean_t: float = 1.6e-4
    quat: float = 1e-3
    scales: float = 5e-3
    opacity: float = 5e-2
    sh: float = 2.5e-3

    def struct(self) -> _capi.Lrs:
        k = _capi.Lrs()
        for n, _ in _capi.Lrs._fields_:
            setattr(k, n, getattr(self, n))
        return k


def _host_scene(scene: HybridScene, dtype) -> tuple[_capi.HostScene, list]:
    hs = _capi.HostScene()
    hs.n4, hs.n3, hs.sh_degree, hs.tau, hs.extent = scene.n4, scene.n3, scene.sh_degree, scene.tau, scene.extent
    hs.duration_seconds = scene.duration_seconds
    keep = []
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        a = np.ascontiguousarray(getattr(scene, f), dtype=dtype)
        keep.append(a)
        setattr(hs, f, ptr(a))
    return hs, keep


def _empty_like_scene(n4: int, n3: int, deg: int, dtype) -> HybridScene:
    K = sh_coeff_count(deg)
    s = HybridScene(sh_degree=deg)
    shapes = dict(mean_x=(n4, 3), mean_t=(n4,), ql=(n4, 4), qr=(n4, 4), log_s4=(n4, 4), op4=(n4,), sh4=(n4, K, 3),
                  mean3=(n3, 3), quat3=(n3, 4), log_s3=(n3, 3), op3=(n3,), sh3=(n3, K, 3))
    for k, shp in shapes.items():
        setattr(s, k, np.zeros(shp, dtype=dtype))
    return s


def _opts(weight_cutoff, num_threads=1, count_map=False, transmittance_map=False) -> _capi.RasterOpts:
    o = _capi.RasterOpts()
    o.weight_cutoff, o.num_threads = weight_cutoff, num_threads
    o.count_map, o.transmittance_map = int(bool(count_map)), int(bool(transmittance_map))
    return o


def _dtype_code(dtype) -> int:
    return HGS_F64 if np.dtype(dtype) == np.float64 else HGS_F32


class Context:
    """One CUDA device: a device-resident scene plus its optimizer state."""

    def __init__(self, device: int = 0):
        self._lib = _capi.lib()
        h = C.c_void_p()
        rc = self._lib.hgs_ctx_create(device, C.byref(h))
        if rc != 0:
            raise CudaError(f"hgs_ctx_create(device={device}) failed with status {rc} (no usable CUDA device?)")
        self._h = h
        self.device = device
        self.sh_degree = 1
        self.n4 = self.n3 = 0
        self._last_shape = (0, 0)

    # ------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.hgs_ctx_destroy(self._h)
            self._h = None

    def __enter__(self) -> "Context":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def __del__(self):
        self.close()

    def _check(self, rc: int) -> None:
        check(self._h, rc)

    @property
    def handle(self):
        return self._h

    def synchronize(self) -> None:
        self._check(self._lib.hgs_synchronize(self._h))

    def set_stream(self, stream_ptr: int | None) -> None:
        self._check(self._lib.hgs_ctx_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    # ------------------------------------------------------------ scene
    def upload(self, scene: HybridScene, dtype=np.float64) -> None:
        scene.validate_shapes()
        hs, keep = _host_scene(scene, dtype)
        self._check(self._lib.hgs_scene_upload(self._h, C.byref(hs), _dtype_code(dtype)))
        self.sh_degree, self.n4, self.n3 = scene.sh_degree, scene.n4, scene.n3
        self._meta = (scene.tau, scene.extent, scene.duration_seconds)
        del keep

    def counts(self) -> tuple[int, int]:
        n4, n3, deg = C.c_int64(), C.c_int64(), C.c_int32()
        self._check(self._lib.hgs_scene_counts(self._h, C.byref(n4), C.byref(n3), C.byref(deg)))
        self.n4, self.n3, self.sh_degree = n4.value, n3.value, deg.value
        return self.n4, self.n3

    def download(self, dtype=np.float64) -> HybridScene:
        n4, n3 = self.counts()
        s = _empty_like_scene(n4, n3, self.sh_degree, dtype)
        hs, keep = _host_scene(s, dtype)
        for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
            setattr(s, f, keep[(HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS).index(f)])
        self._check(self._lib.hgs_scene_download(self._h, C.byref(hs), _dtype_code(dtype)))
        s.tau, s.extent, s.duration_seconds = hs.tau, hs.extent, hs.duration_seconds
        return s

    # ------------------------------------------------------------ multi-GPU exchange
    @staticmethod
    def comm_unique_id() -> bytes:
        """ncclGetUniqueId (128 bytes) -- on one rank, shipped out of band."""
        k = _capi.CommId()
        rc = _capi.lib().hgs_comm_unique_id(C.byref(k))
        if rc != 0:
            raise _capi.CudaError("comm: NCCL unavailable")
        return bytes(C.string_at(C.addressof(k), 128))

    def comm_init(self, nranks: int, rank: int, uid: bytes) -> None:
        k = _capi.CommId()
        C.memmove(C.addressof(k), uid, 128)
        self._check(self._lib.hgs_comm_init(self._h, int(nranks), int(rank), C.byref(k)))
        self._comm_world = int(nranks)

    def comm_destroy(self) -> None:
        self._check(self._lib.hgs_comm_destroy(self._h))
        self._comm_world = None

    def allreduce_grads(self) -> None:
        """Sum the packed gradient payload over the ranks (stream-ordered)."""
        self._check(self._lib.hgs_allreduce_grads(self._h))

    def allreduce_f64(self, vals) -> np.ndarray:
        a = np.ascontiguousarray(vals, dtype=np.float64).copy()
        self._check(self._lib.hgs_allreduce_f64(self._h, a.ctypes.data_as(_capi._dp), a.size))
        return a

    def param_checksum(self) -> int:
        """Order-independent 64-bit checksum of the parameters."""
        v = C.c_uint64()
        self._check(self._lib.hgs_param_checksum(self._h, C.byref(v)))
        return v.value

    def broadcast_params(self, root: int = 0) -> None:
        self._check(self._lib.hgs_broadcast_params(self._h, int(root)))

    def set_sharded(self, enable: bool = True) -> None:
        """Sharded optimizer exchange for train_exchange_async: reduce-scatter
        of the gradient rows, Adam on this rank's shard, all-gather of the
        parameters (hgs_comm_set_sharded)."""
        self._check(self._lib.hgs_comm_set_sharded(self._h, 1 if enable else 0))

    def gather_state(self) -> None:
        """Whole Adam moments on every rank (collective; a no-op unless the
        sharded exchange left them sharded)."""
        self._check(self._lib.hgs_gather_state(self._h))

    @staticmethod
    def shard_range(n: int, ranks: int, rank: int) -> tuple[int, int]:
        lo, hi = C.c_int64(), C.c_int64()
        _capi.lib().hgs_shard_range(int(n), int(ranks), int(rank), C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    # ------------------------------------------------------------ initialisation
    def init_scene(self, positions: np.ndarray, rgb: np.ndarray, cfg: "InitConfig | None" = None) -> None:
        """init_scene (data_io.cpp:189-238) straight into the device: one
        dynamic Gaussian per point, the 3-NN scales from a GPU kNN."""
        cfg = cfg or InitConfig()
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        col = np.ascontiguousarray(rgb, dtype=np.float64).reshape(-1, 3)
        if pos.shape != col.shape:
            raise ValueError("init_scene: positions and rgb differ in length")
        self._check(self._lib.hgs_init_scene(self._h, pos.ctypes.data_as(_capi._dp), col.ctypes.data_as(_capi._dp),
                                             pos.shape[0], C.byref(cfg.struct())))
        self.counts()

    # ------------------------------------------------------------ checkpoints
    def save_checkpoint(self, path: str, with_state: bool = True) -> None:
        """save_checkpoint (data_io.cpp:656-665) of the device scene and, with
        ``with_state``, its optimizer state -- encoded on the device."""
        self._check(self._lib.hgs_checkpoint_save(self._h, os.fsencode(path), int(bool(with_state))))

    def load_checkpoint(self, path: str) -> bool:
        """load_checkpoint (data_io.cpp:667-719) into the device; returns
        whether the file carried optimizer state (else it is zeroed)."""
        has = C.c_int()
        self._check(self._lib.hgs_checkpoint_load(self._h, os.fsencode(path), C.byref(has)))
        self.counts()
        return bool(has.value)

    # ------------------------------------------------------------ render
    def render(self, camera: Camera, t: float, background=(0.0, 0.0, 0.0), weight_cutoff=DEFAULT_WEIGHT_CUTOFF,
               count_map=False, transmittance_map=False) -> dict:
        H, W = camera.height, camera.width
        rgb = np.empty((H, W, 3), dtype=np.float32)
        counts = np.empty((H, W), dtype=np.uint32) if count_map else None
        trans = np.empty((H, W), dtype=np.float32) if transmittance_map else None
        st = _capi.RenderStats()
        bg = np.ascontiguousarray(background, dtype=np.float64)
        o = _opts(weight_cutoff, 1, count_map, transmittance_map)
        self._check(self._lib.hgs_render(self._h, C.byref(_capi.camera_struct(camera)), float(t),
                                         bg.ctypes.data_as(_capi._dp), C.byref(o),
                                         rgb.ctypes.data_as(_capi._fp),
                                         counts.ctypes.data_as(_capi._u32p) if counts is not None else None,
                                         trans.ctypes.data_as(_capi._fp) if trans is not None else None,
                                         C.byref(st)))
        self._last_shape = (H, W)
        return {"rgb": rgb, "counts": counts, "transmittance": trans,
                "stats": {n: int(getattr(st, n)) for n, _ in _capi.RenderStats._fields_}}

    def render_sweep(self, cameras: list, times: list, background=(0.0, 0.0, 0.0),
                     weight_cutoff=DEFAULT_WEIGHT_CUTOFF, out=None, with_stats: bool = False):
        """Render n frames (cameras[f], times[f]) with one synchronisation
        (hgs_render_sweep; the c5 render sweep).  out: None (no image
        output, e.g. timing), "host" (returns an (n, h, w, 3) float32
        array) or a CUDA tensor / device pointer of n*h*w*3 floats."""
        n = len(cameras)
        cams = (_capi.Camera_ * max(1, n))(*[_capi.camera_struct(c) for c in cameras])
        ts = (C.c_double * max(1, n))(*[float(t) for t in times])
        bg = np.ascontiguousarray(background, dtype=np.float64)
        o = _opts(weight_cutoff)
        st = (_capi.RenderStats * max(1, n))() if with_stats else None
        host = None
        ptr_out, on_dev = None, 0
        if isinstance(out, str) and out == "host":
            h, w = cameras[0].height, cameras[0].width
            host = np.empty((n, h, w, 3), dtype=np.float32)
            ptr_out = host.ctypes.data_as(_capi._fp)
        elif out is not None:
            addr = out.data_ptr() if hasattr(out, "data_ptr") else int(out)
            ptr_out, on_dev = C.cast(C.c_void_p(addr), _capi._fp), 1
        self._check(self._lib.hgs_render_sweep(self._h, n, cams, ts, bg.ctypes.data_as(_capi._dp), C.byref(o),
                                               ptr_out, on_dev, st))
        if n:
            self._last_shape = (cameras[-1].height, cameras[-1].width)
        stats = [{k: int(getattr(x, k)) for k, _ in _capi.RenderStats._fields_} for x in st[:n]] if with_stats else None
        res = host if host is not None else out
        return (res, stats) if with_stats else res

    def render_device(self, camera: Camera, t: float, background=(0.0, 0.0, 0.0),
                      weight_cutoff=DEFAULT_WEIGHT_CUTOFF) -> None:
        """Render into the context's device image only (no host copy); read
        it with last_image_device_ptr() or score it with image_metrics()."""
        bg = np.ascontiguousarray(background, dtype=np.float64)
        o = _opts(weight_cutoff)
        self._check(self._lib.hgs_render(self._h, C.byref(_capi.camera_struct(camera)), float(t),
                                         bg.ctypes.data_as(_capi._dp), C.byref(o), None, None, None, None))
        self._last_shape = (camera.height, camera.width)

    def image_metrics(self, gt: np.ndarray | None = None, gt_device_ptr: int | None = None,
                      gt_u8: bool = False, want_ssim: bool = True) -> tuple[float, float | None]:
        """(psnr, ssim) of the last rendered image against gt (metrics.cpp:91-101
        and the valid-window SSIM), on the device.  gt: (h, w, 3) float64 /
        float32 linear, or uint8 sRGB; or a device float32 / uint8 frame."""
        p, q = C.c_double(), C.c_double()
        qs = C.byref(q) if want_ssim else None
        if gt_device_ptr is not None:
            self._check(self._lib.hgs_image_metrics(self._h, C.c_void_p(gt_device_ptr), HGS_U8 if gt_u8 else HGS_F32,
                                                    1, C.byref(p), qs))
        else:
            a = np.ascontiguousarray(gt)
            if a.shape != self._last_shape + (3,):
                raise ValueError("metrics: image dimensions differ")
            if a.dtype == np.uint8:
                code = HGS_U8
            else:
                code = _dtype_code(a.dtype)
                a = a.astype(np.float64 if code == HGS_F64 else np.float32, copy=False)
            self._check(self._lib.hgs_image_metrics(self._h, ptr(a), code, 0, C.byref(p), qs))
        return p.value, (q.value if want_ssim else None)

    def density_map(self, camera: Camera, t: float, dynamics_only: bool = False,
                    weight_cutoff: float = DEFAULT_WEIGHT_CUTOFF) -> np.ndarray:
        """raster.cpp:268-287 on the device: (h, w) uint32 splat coverage
        counts of the resident scene.  Releases the last render's tape."""
        out = np.empty((camera.height, camera.width), dtype=np.uint32)
        self._check(self._lib.hgs_density_map(self._h, C.byref(_capi.camera_struct(camera)), float(t),
                                              int(bool(dynamics_only)), float(weight_cutoff),
                                              out.ctypes.data_as(_capi._u32p)))
        return out

    def render_info(self) -> dict:
        info = _capi.RenderInfo()
        self._check(self._lib.hgs_render_info_get(self._h, C.byref(info)))
        return {n: int(getattr(info, n)) for n, _ in _capi.RenderInfo._fields_}

    def last_image_device_ptr(self) -> int:
        return int(self._lib.hgs_last_image_device(self._h) or 0)

    # ------------------------------------------------------------ parity introspection
    def debug_splats(self) -> dict:
        n = C.c_int64()
        self._check(self._lib.hgs_debug_splats(self._h, None, None, None, None, None, None, None, 0, C.byref(n)))
        V = n.value
        out = dict(gid=np.zeros(V, np.int32), depth_bits=np.zeros(V, np.uint32), box=np.zeros((V, 4), np.int32),
                   mean=np.zeros((V, 2)), conic=np.zeros((V, 4)), alpha=np.zeros(V), rgb=np.zeros((V, 3), np.float32))
        if V:
            self._check(self._lib.hgs_debug_splats(
                self._h, out["gid"].ctypes.data_as(_capi._i32p), out["depth_bits"].ctypes.data_as(_capi._u32p),
                out["box"].ctypes.data_as(_capi._i32p), out["mean"].ctypes.data_as(_capi._dp),
                out["conic"].ctypes.data_as(_capi._dp), out["alpha"].ctypes.data_as(_capi._dp),
                out["rgb"].ctypes.data_as(_capi._fp), V, C.byref(n)))
        return out

    def debug_keep_instances(self, enable: bool = True) -> None:
        self._check(self._lib.hgs_debug_keep_instances(self._h, int(enable)))

    def debug_instances(self) -> tuple[np.ndarray, np.ndarray]:
        n = C.c_int64()
        self._check(self._lib.hgs_debug_instances(self._h, None, None, 0, C.byref(n)))
        tile = np.zeros(n.value, np.uint32)
        gid = np.zeros(n.value, np.uint32)
        if n.value:
            self._check(self._lib.hgs_debug_instances(self._h, tile.ctypes.data_as(_capi._u32p),
                                                      gid.ctypes.data_as(_capi._u32p), n.value, C.byref(n)))
        return tile, gid

    def debug_instance_masks(self) -> np.ndarray:
        """Quadrant masks of the kept full instance list (debug_instances order)."""
        n = C.c_int64()
        self._check(self._lib.hgs_debug_instance_masks(self._h, None, 0, C.byref(n)))
        m = np.zeros(n.value, np.uint8)
        if n.value:
            self._check(self._lib.hgs_debug_instance_masks(self._h, m.ctypes.data_as(C.POINTER(C.c_uint8)), n.value,
                                                           C.byref(n)))
        return m

    # ------------------------------------------------------------ training
    def forward_train(self, camera: Camera, t: float, background=(0.0, 0.0, 0.0),
                      weight_cutoff=DEFAULT_WEIGHT_CUTOFF, want_image=True) -> np.ndarray | None:
        H, W = camera.height, camera.width
        rgb = np.empty((H, W, 3), dtype=np.float32) if want_image else None
        bg = np.ascontiguousarray(background, dtype=np.float64)
        o = _opts(weight_cutoff)
        self._check(self._lib.hgs_forward_train(self._h, C.byref(_capi.camera_struct(camera)), float(t),
                                                bg.ctypes.data_as(_capi._dp), C.byref(o),
                                                rgb.ctypes.data_as(_capi._fp) if rgb is not None else None))
        self._last_shape = (H, W)
        return rgb

    def backward(self, loss_grad: np.ndarray | None = None, scale: float = 1.0) -> None:
        """Accumulate scale * dL/dparams; loss_grad None = use the device
        gradient left by :meth:`loss_with_grad`."""
        if loss_grad is None:
            self._check(self._lib.hgs_backward(self._h, None, HGS_F32, 1, float(scale)))
            return
        g = np.ascontiguousarray(loss_grad)
        code = _dtype_code(g.dtype)
        g = g.astype(np.float64 if code == HGS_F64 else np.float32, copy=False)
        self._check(self._lib.hgs_backward(self._h, ptr(g), code, 0, float(scale)))

    def set_exact_backward(self, enable: bool = True) -> None:
        """FP64 pair terms for every pixel in backward() / training (the
        reference's arithmetic; several times slower than the default)."""
        self._check(self._lib.hgs_set_exact_backward(self._h, 1 if enable else 0))

    def zero_grads(self) -> None:
        self._check(self._lib.hgs_zero_grads(self._h))

    def grads(self, dtype=np.float64) -> dict:
        n4, n3 = self.counts()
        s = _empty_like_scene(n4, n3, self.sh_degree, dtype)
        hs, keep = _host_scene(s, dtype)
        sn4 = np.zeros(n4, dtype=dtype)
        sn3 = np.zeros(n3, dtype=dtype)
        self._check(self._lib.hgs_grads_download(self._h, C.byref(hs), _dtype_code(dtype), ptr(sn4), ptr(sn3)))
        out = {f: keep[i] for i, f in enumerate(HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS)}
        out["screen_norm4"], out["screen_norm3"] = sn4, sn3
        return out

    def upload_grads(self, grads: dict, dtype=np.float64) -> None:
        """Host gradients (the fields of grads(), same shapes) into the device
        gradient rows (hgs_grads_upload) -- the optimizer_step(scene, const
        SceneGrads&, ...) entry of train.hpp:68-69 with host gradients."""
        n4, n3 = self.counts()
        s = _empty_like_scene(n4, n3, self.sh_degree, dtype)
        for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
            a = np.ascontiguousarray(grads[f], dtype=dtype)
            if a.shape != getattr(s, f).shape:
                raise ValueError(f"gradient {f}: shape {a.shape}, expected {getattr(s, f).shape}")
            setattr(s, f, a)
        hs, keep = _host_scene(s, dtype)
        self._check(self._lib.hgs_grads_upload(self._h, C.byref(hs), _dtype_code(dtype)))
        del keep

    def grads_packed(self) -> tuple[int, int]:
        """(device pointer, float count) of the packed gradient payload
        (hgs_grads_packed): valid gradient rows + stat deltas, contiguous."""
        p, n = _capi._fp(), C.c_int64()
        self._check(self._lib.hgs_grads_packed(self._h, 0, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value or 0, n.value

    def grads_unpack(self) -> None:
        """Scatter the (reduced) packed payload back into the gradient rows."""
        self._check(self._lib.hgs_grads_packed(self._h, 1, None, None))

    def grads_device(self) -> tuple[int, int]:
        p = _capi._fp()
        n = C.c_int64()
        self._check(self._lib.hgs_grads_device(self._h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value or 0, n.value

    def loss_with_grad(self, gt: np.ndarray | None = None, ssim_lambda: float = 0.2, gt_device_ptr: int | None = None,
                       want_grad: bool = False):
        loss = C.c_double()
        g_out = None
        if gt_device_ptr is not None:
            g_out = np.empty(self._last_shape + (3,), dtype=np.float32) if want_grad else None
            self._check(self._lib.hgs_loss_with_grad(self._h, C.c_void_p(gt_device_ptr), HGS_F32, 1,
                                                     float(ssim_lambda), C.byref(loss), ptr(g_out)))
        else:
            a = np.ascontiguousarray(gt)
            code = _dtype_code(a.dtype)
            a = a.astype(np.float64 if code == HGS_F64 else np.float32, copy=False)
            if a.shape != self._last_shape + (3,):
                raise ValueError("photometric_loss: image dimensions differ")
            g_out = np.empty(a.shape, dtype=a.dtype) if want_grad else None  # same dtype as gt (C ABI)
            self._check(self._lib.hgs_loss_with_grad(self._h, ptr(a), code, 0, float(ssim_lambda), C.byref(loss),
                                                     ptr(g_out)))
        return (loss.value, g_out) if want_grad else loss.value

    def adam_step(self, lrs: LearningRates | None = None, mean_lr_scale: float = 1.0) -> int:
        sk = C.c_int64()
        self._check(self._lib.hgs_adam_step(self._h, C.byref((lrs or LearningRates()).struct()),
                                            float(mean_lr_scale), C.byref(sk)))
        return sk.value

    def adam_state(self, dtype=np.float64):
        n4, n3 = self.counts()
        m = _empty_like_scene(n4, n3, self.sh_degree, dtype)
        v = _empty_like_scene(n4, n3, self.sh_degree, dtype)
        hm, km = _host_scene(m, dtype)
        hv, kv = _host_scene(v, dtype)
        step = C.c_uint64()
        self._check(self._lib.hgs_adam_state_download(self._h, C.byref(hm), C.byref(hv), _dtype_code(dtype),
                                                      C.byref(step)))
        F = HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS
        for i, f in enumerate(F):
            setattr(m, f, km[i])
            setattr(v, f, kv[i])
        return m, v, step.value

    def set_adam_state(self, m: HybridScene, v: HybridScene, step: int, dtype=np.float64) -> None:
        hm, km = _host_scene(m, dtype)
        hv, kv = _host_scene(v, dtype)
        self._check(self._lib.hgs_adam_state_upload(self._h, C.byref(hm), C.byref(hv), _dtype_code(dtype), step))

    def densify_stats(self):
        n4, n3 = self.counts()
        gn4, gn3 = np.zeros(n4), np.zeros(n3)
        c4, c3 = np.zeros(n4, np.uint32), np.zeros(n3, np.uint32)
        self._check(self._lib.hgs_stats_download(self._h, gn4.ctypes.data_as(_capi._dp),
                                                 c4.ctypes.data_as(_capi._u32p), gn3.ctypes.data_as(_capi._dp),
                                                 c3.ctypes.data_as(_capi._u32p)))
        return gn4, c4, gn3, c3

    def densify_and_prune(self, rng, grad_threshold: float = 0.02, opacity_prune_eps: float = 0.005,
                          clone_size_frac: float = 0.01, split_factor: float = 1.6,
                          max_gaussians: int = 20000) -> dict:
        """densify_and_prune (train.cpp:182-299) on the device; ``rng`` is the
        loop's rng.MT19937_64, advanced exactly like the reference's."""
        cfg = _capi.DensifyCfg(grad_threshold, opacity_prune_eps, clone_size_frac, split_factor, max_gaussians)
        if isinstance(rng, Rng):  # native stream: one C call (plan, draws, apply)
            rep = _capi.DensifyReport()
            self._check(self._lib.hgs_densify_and_prune(self._h, C.byref(cfg), rng.handle, C.byref(rep)))
            self.counts()
            return {n: int(getattr(rep, n)) for n, _ in _capi.DensifyReport._fields_}
        from .rng import densify_normals

        n4, n3 = self.counts()
        k3, k4 = np.zeros(max(n3, 1), np.uint8), np.zeros(max(n4, 1), np.uint8)
        rep = _capi.DensifyReport()
        self._check(self._lib.hgs_densify_plan(self._h, C.byref(cfg), k3.ctypes.data_as(C.c_void_p),
                                               k4.ctypes.data_as(C.c_void_p), C.byref(rep)))
        d3 = rep.cloned3 + rep.split3
        d4 = rep.cloned4 + rep.split4
        nrm3, nrm4 = densify_normals(rng, k3[:d3].tolist(), k4[:d4].tolist())
        self._check(self._lib.hgs_densify_apply(self._h, nrm3.ctypes.data_as(_capi._dp),
                                                nrm4.ctypes.data_as(_capi._dp), float(split_factor)))
        self.counts()
        return {n: int(getattr(rep, n)) for n, _ in _capi.DensifyReport._fields_}

    def opacity_reset(self, floor_logit: float | None = None) -> None:
        """train.cpp:459-465: opacity logits capped at logit(0.01)."""
        import math

        f = math.log(0.01 / 0.99) if floor_logit is None else floor_logit
        self._check(self._lib.hgs_opacity_reset(self._h, float(f)))

    def sweep_convert(self):
        n4, _ = self.counts()
        moved = np.zeros(max(n4, 1), dtype=np.int64)
        rep = _capi.ConversionReport()
        self._check(self._lib.hgs_sweep_convert(self._h, moved.ctypes.data_as(_capi._i64p), C.byref(rep)))
        self.counts()
        return moved[: rep.count].copy(), {"count": int(rep.count), "max_leakage": rep.max_leakage,
                                           "mean_leakage": rep.mean_leakage}


class Rng:
    """The training loop's random stream (hgs_rng: libstdc++ std::mt19937_64
    with the reference's distributions, train.cpp:68-72, 245-275, 387-404)."""

    def __init__(self, seed: int = 5489):
        self._lib = _capi.lib()
        h = _capi._vp()
        if self._lib.hgs_rng_create(C.c_uint64(seed), C.byref(h)) != 0:
            raise MemoryError("hgs_rng_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.hgs_rng_destroy(self._h)
            self._h = None

    def raw(self) -> int:
        return int(self._lib.hgs_rng_raw(self._h))

    def index(self, lo: int, hi: int) -> int:
        """std::uniform_int_distribution<size_t>(lo, hi)"""
        return int(self._lib.hgs_rng_index(self._h, lo, hi))

    def batch(self, n_samples: int, count: int) -> list[int]:
        """`count` picks over [0, n_samples - 1] (train.cpp:403-404)."""
        out = (C.c_uint64 * max(1, count))()
        if self._lib.hgs_rng_batch(self._h, n_samples, count, out) != 0:
            raise ValueError("rng batch: bad arguments")
        return [int(v) for v in out[:count]]

    def densify_normals(self, kinds3, kinds4):
        """The normals densify_and_prune draws (hgs_densify_normals)."""
        k3 = np.ascontiguousarray(kinds3, dtype=np.uint8)
        k4 = np.ascontiguousarray(kinds4, dtype=np.uint8)
        n3, n4 = np.zeros(6 * max(1, k3.size)), np.zeros(8 * max(1, k4.size))
        rc = self._lib.hgs_densify_normals(self._h, k3.ctypes.data_as(C.c_void_p), k3.size,
                                           k4.ctypes.data_as(C.c_void_p), k4.size, n3.ctypes.data_as(_capi._dp),
                                           n4.ctypes.data_as(_capi._dp))
        if rc != 0:
            raise ValueError("densify_normals: bad arguments")
        return n3, n4


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def rasterize(scene: HybridScene, camera: Camera, t: float, background=(0.0, 0.0, 0.0), num_threads: int = 1,
              weight_cutoff: float = DEFAULT_WEIGHT_CUTOFF, count_map: bool = False,
              transmittance_map: bool = False, full: bool = False):
    """hybridgs.rasterize (bindings.cpp:147-155): (h, w, 3) float64 image.

    Literal drop-in (host scene in, host image out) through hgs_rasterize.
    ``full=True`` returns the RenderOutput-like dict with counts/transmittance
    and RenderStats (raster.hpp:49-54).
    """
    ctx = default_context()
    hs, keep = _host_scene(scene, np.float64)
    H, W = camera.height, camera.width
    rgb = np.empty((H, W, 3), dtype=np.float64)
    counts = np.empty((H, W), dtype=np.uint32) if count_map else None
    trans = np.empty((H, W), dtype=np.float64) if transmittance_map else None
    st = _capi.RenderStats()
    bg = np.ascontiguousarray(background, dtype=np.float64)
    o = _opts(weight_cutoff, num_threads, count_map, transmittance_map)
    ctx._check(ctx._lib.hgs_rasterize(ctx.handle, C.byref(hs), HGS_F64, C.byref(_capi.camera_struct(camera)),
                                      float(t), bg.ctypes.data_as(_capi._dp), C.byref(o), ptr(rgb),
                                      counts.ctypes.data_as(_capi._u32p) if counts is not None else None,
                                      ptr(trans), C.byref(st)))
    ctx.sh_degree, ctx.n4, ctx.n3 = scene.sh_degree, scene.n4, scene.n3
    del keep
    if not full:
        return rgb
    return {"rgb": rgb, "counts": counts, "transmittance": trans,
            "stats": {n: int(getattr(st, n)) for n, _ in _capi.RenderStats._fields_}}


def density_map(scene: HybridScene, camera: Camera, t: float, dynamics_only: bool = False,
                weight_cutoff: float = DEFAULT_WEIGHT_CUTOFF) -> np.ndarray:
    """hybridgs.density_map (bindings.cpp:165-172): (h, w) uint32 counts."""
    ctx = default_context()
    ctx.upload(scene)
    return ctx.density_map(camera, t, dynamics_only, weight_cutoff)


def sweep_convert(scene: HybridScene) -> tuple[int, float, float]:
    """hybridgs.sweep_convert (bindings.cpp:135-138; scene.cpp:43-71): converts
    every dynamic Gaussian with exp(s_t) > tau to a static one IN PLACE (on
    the device) and returns (count, max_leakage, mean_leakage)."""
    ctx = default_context()
    ctx.upload(scene)
    _, rep = ctx.sweep_convert()
    out = ctx.download()
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS + ("tau", "extent", "duration_seconds"):
        setattr(scene, f, getattr(out, f))
    return rep["count"], rep["max_leakage"], rep["mean_leakage"]


def _metrics(a: np.ndarray, b: np.ndarray, want_psnr: bool, want_ssim: bool) -> tuple[float, float]:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("metrics: image dimensions differ")
    ctx = default_context()
    p, q = C.c_double(), C.c_double()
    ctx._check(ctx._lib.hgs_metrics(ctx.handle, ptr(a), ptr(b), HGS_F64, a.shape[1], a.shape[0],
                                    C.byref(p) if want_psnr else None, C.byref(q) if want_ssim else None))
    return p.value, q.value


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """hybridgs.psnr (metrics.cpp:91-101) on the device: 10 log10(1 / MSE)."""
    return _metrics(a, b, True, False)[0]


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    """hybridgs.ssim (metrics.cpp): mean SSIM over the valid 11x11 windows."""
    return _metrics(a, b, False, True)[1]


@dataclass
class InitConfig:  # data_io.hpp:43-49
    sh_degree: int = 1
    tau: float = 0.5
    duration_seconds: float = 1.0
    init_temporal_scale: float = 0.1
    init_opacity: float = 0.1

    def struct(self) -> _capi.InitCfg:
        k = _capi.InitCfg()
        k.sh_degree, k.tau, k.duration_seconds = int(self.sh_degree), float(self.tau), float(self.duration_seconds)
        k.init_temporal_scale, k.init_opacity = float(self.init_temporal_scale), float(self.init_opacity)
        return k


def init_scene(points, cfg: InitConfig | None = None, ctx: "Context | None" = None) -> HybridScene:
    """hgs::init_scene (data_io.cpp:189-238): ``points`` is a
    dataset.InitPoints or a (positions, rgb) pair; returns the host scene
    (the device copy stays resident in ``ctx``)."""
    pos, rgb = (points.positions, points.rgb) if hasattr(points, "positions") else points
    ctx = ctx or default_context()
    ctx.init_scene(pos, rgb, cfg)
    return ctx.download()


@dataclass
class CheckpointState:
    """GradAccum (optim.hpp:32-41): Adam moments shaped like the scene,
    densification statistics and the step / skipped-row counters."""
    m: HybridScene
    v: HybridScene
    grad_norm4: np.ndarray
    grad_norm3: np.ndarray
    count4: np.ndarray
    count3: np.ndarray
    step: int = 0
    skipped_nonfinite: int = 0

    @staticmethod
    def zeros_like(scene: HybridScene) -> "CheckpointState":
        z = lambda: _empty_like_scene(scene.n4, scene.n3, scene.sh_degree, np.float64)  # noqa: E731
        return CheckpointState(z(), z(), np.zeros(scene.n4), np.zeros(scene.n3), np.zeros(scene.n4, np.uint32),
                               np.zeros(scene.n3, np.uint32))


def _host_state(st: CheckpointState) -> tuple[_capi.HostState, list]:
    hs = _capi.HostState()
    hs.step, hs.skipped_nonfinite = int(st.step), int(st.skipped_nonfinite)
    hm, km = _host_scene(st.m, np.float64)
    hv, kv = _host_scene(st.v, np.float64)
    hs.m, hs.v = hm, hv
    arrs = [np.ascontiguousarray(st.grad_norm4, np.float64), np.ascontiguousarray(st.grad_norm3, np.float64),
            np.ascontiguousarray(st.count4, np.uint32), np.ascontiguousarray(st.count3, np.uint32)]
    hs.grad_norm4, hs.grad_norm3 = arrs[0].ctypes.data_as(_capi._dp), arrs[1].ctypes.data_as(_capi._dp)
    hs.count4, hs.count3 = arrs[2].ctypes.data_as(_capi._u32p), arrs[3].ctypes.data_as(_capi._u32p)
    return hs, [km, kv, arrs]


def save_checkpoint(scene: HybridScene, path: str, state: CheckpointState | None = None) -> None:
    """hybridgs.save_checkpoint (bindings.cpp:197-201; data_io.cpp:656-665):
    a host scene in double precision, byte-identical to the reference."""
    lib = _capi.lib()
    hs, keep = _host_scene(scene, np.float64)
    st, keep2 = _host_state(state) if state is not None else (None, None)
    check_io(lib.hgs_checkpoint_write(C.byref(hs), C.byref(st) if st is not None else None, os.fsencode(path)))
    del keep, keep2


def load_checkpoint_full(path: str) -> tuple[HybridScene, CheckpointState | None]:
    """load_checkpoint (data_io.cpp:667-719): (scene, state or None)."""
    lib = _capi.lib()
    n4, n3, deg, has = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int()
    p = os.fsencode(path)
    check_io(lib.hgs_checkpoint_info(p, C.byref(n4), C.byref(n3), C.byref(deg), C.byref(has)))
    scene = _empty_like_scene(n4.value, n3.value, deg.value, np.float64)
    hs, keep = _host_scene(scene, np.float64)
    for i, f in enumerate(HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS):
        setattr(scene, f, keep[i])
    state = CheckpointState.zeros_like(scene) if has.value else None
    st, keep2 = _host_state(state) if state is not None else (None, None)
    check_io(lib.hgs_checkpoint_read(p, C.byref(hs), C.byref(st) if st is not None else None))
    scene.tau, scene.extent, scene.duration_seconds = hs.tau, hs.extent, hs.duration_seconds
    if state is not None:
        km, kv, arrs = keep2
        for i, f in enumerate(HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS):
            setattr(state.m, f, km[i])
            setattr(state.v, f, kv[i])
        state.grad_norm4, state.grad_norm3, state.count4, state.count3 = arrs
        state.step, state.skipped_nonfinite = int(st.step), int(st.skipped_nonfinite)
    return scene, state


def load_checkpoint(path: str) -> HybridScene:
    """hybridgs.load_checkpoint (bindings.cpp:202-205): the scene."""
    return load_checkpoint_full(path)[0]
