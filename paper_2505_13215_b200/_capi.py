"""ctypes binding of libhgs_gpu.so (include/hgs_gpu.h).

This is the reference-side binding a maintainer would add:
plain ctypes over the C ABI.  There is no fallback: if the library or a CUDA
device is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGS_LIB") or os.path.join(_HERE, "libhgs_gpu.so")  # HGS_LIB: A/B builds

HGS_F64, HGS_F32, HGS_U8 = 0, 1, 2

_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class HostScene(C.Structure):
    _fields_ = [("n4", C.c_int64), ("n3", C.c_int64), ("sh_degree", C.c_int32), ("tau", C.c_double),
                ("extent", C.c_double)] + [(n, _vp) for n in ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4",
                                                              "sh4", "mean3", "quat3", "log_s3", "op3", "sh3")] + \
        [("duration_seconds", C.c_double)]


class CommId(C.Structure):  # hgs_comm_id (ncclUniqueId)
    _fields_ = [("internal", C.c_char * 128)]


class InitCfg(C.Structure):  # hgs_init_cfg (InitConfig, data_io.hpp:43-49)
    _fields_ = [("sh_degree", C.c_int32), ("tau", C.c_double), ("duration_seconds", C.c_double),
                ("init_temporal_scale", C.c_double), ("init_opacity", C.c_double)]


class HostState(C.Structure):  # hgs_host_state (GradAccum, optim.hpp:32-41)
    _fields_ = [("step", C.c_uint64), ("skipped_nonfinite", C.c_uint64), ("m", HostScene), ("v", HostScene),
                ("grad_norm4", _dp), ("grad_norm3", _dp), ("count4", _u32p), ("count3", _u32p)]


class Camera_(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("rot", C.c_double * 9), ("trans", C.c_double * 3), ("width", C.c_int32), ("height", C.c_int32),
                ("near_", C.c_double), ("far_", C.c_double)]


class RenderStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("culled_depth", "culled_offscreen", "culled_degenerate",
                                         "culled_temporal", "degenerate_temporal", "projected")]


class RasterOpts(C.Structure):
    _fields_ = [("weight_cutoff", C.c_double), ("num_threads", C.c_int32), ("count_map", C.c_int32),
                ("transmittance_map", C.c_int32)]


class Lrs(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mean", "mean_final_ratio", "mean_t", "quat", "scales", "opacity", "sh")]


class ConversionReport(C.Structure):
    _fields_ = [("count", C.c_int64), ("max_leakage", C.c_double), ("mean_leakage", C.c_double)]


class RenderInfo(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("visible", "instances", "fixup_pixels", "kept_instances",
                                         "sweep_redone_frames")]


class TrainOpts(C.Structure):
    _fields_ = [("ssim_lambda", C.c_double), ("weight_cutoff", C.c_double), ("mean_lr_scale", C.c_double),
                ("lrs", Lrs), ("bg", C.c_double * 3)]


class DensifyCfg(C.Structure):
    _fields_ = [("grad_threshold", C.c_double), ("opacity_prune_eps", C.c_double),
                ("clone_size_frac", C.c_double), ("split_factor", C.c_double), ("max_gaussians", C.c_int64)]


class DensifyReport(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("cloned3", "split3", "pruned3", "cloned4", "split4", "pruned4",
                                         "new_n3", "new_n4")]


class HgsError(RuntimeError):
    """Base of the errors raised from hgs_status codes."""


class DegenerateTemporalError(HgsError):
    pass


class DegenerateRotationError(HgsError):
    pass


class NumericAbort(HgsError):
    pass


class CudaError(HgsError):
    pass


class FormatError(HgsError):  # errors.hpp FormatError
    pass


class IntegrityError(HgsError):  # errors.hpp IntegrityError
    pass


class UnsupportedVersionError(HgsError):  # errors.hpp UnsupportedVersionError
    pass


class StateError(HgsError):
    pass


_STATUS = {1: ValueError, 2: DegenerateTemporalError, 3: DegenerateRotationError, 4: NumericAbort, 5: CudaError,
           6: StateError, 7: FormatError, 8: IntegrityError, 9: UnsupportedVersionError}

_SIGS = {
    "hgs_ctx_create": ([C.c_int, C.POINTER(_vp)], C.c_int),
    "hgs_ctx_destroy": ([_vp], None),
    "hgs_last_error": ([_vp], C.c_char_p),
    "hgs_ctx_set_stream": ([_vp, _vp], C.c_int),
    "hgs_ctx_stream": ([_vp], _vp),
    "hgs_synchronize": ([_vp], C.c_int),
    "hgs_scene_upload": ([_vp, C.POINTER(HostScene), C.c_int], C.c_int),
    "hgs_scene_download": ([_vp, C.POINTER(HostScene), C.c_int], C.c_int),
    "hgs_scene_counts": ([_vp, _i64p, _i64p, _i32p], C.c_int),
    "hgs_rasterize": ([_vp, C.POINTER(HostScene), C.c_int, C.POINTER(Camera_), C.c_double, _dp,
                       C.POINTER(RasterOpts), _vp, _u32p, _vp, C.POINTER(RenderStats)], C.c_int),
    "hgs_render": ([_vp, C.POINTER(Camera_), C.c_double, _dp, C.POINTER(RasterOpts), _fp, _u32p, _fp,
                    C.POINTER(RenderStats)], C.c_int),
    "hgs_last_image_device": ([_vp], _vp),
    "hgs_render_info_get": ([_vp, C.POINTER(RenderInfo)], C.c_int),
    "hgs_set_exact_backward": ([_vp, C.c_int], C.c_int),
    "hgs_debug_set_sweep_capacity": ([_vp, C.c_int64], C.c_int),
    "hgs_skipped_nonfinite": ([_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], C.c_int),
    "hgs_grads_upload": ([_vp, C.POINTER(HostScene), C.c_int], C.c_int),
    "hgs_stats_upload": ([_vp, _dp, _u32p, _dp, _u32p], C.c_int),
    "hgs_debug_splats": ([_vp, _i32p, _u32p, _i32p, _dp, _dp, _dp, _fp, C.c_int64, _i64p], C.c_int),
    "hgs_debug_instances": ([_vp, _u32p, _u32p, C.c_int64, _i64p], C.c_int),
    "hgs_debug_keep_instances": ([_vp, C.c_int], C.c_int),
    "hgs_debug_pair_counters": ([_vp, C.POINTER(C.c_ulonglong), C.c_int], C.c_int),
    "hgs_comm_set_sharded": ([_vp, C.c_int], C.c_int),
    "hgs_gather_state": ([_vp], C.c_int),
    "hgs_shard_range": ([C.c_int64, C.c_int, C.c_int, _i64p, _i64p], None),
    "hgs_debug_instance_masks": ([_vp, C.POINTER(C.c_uint8), C.c_int64, _i64p], C.c_int),
    "hgs_forward_train": ([_vp, C.POINTER(Camera_), C.c_double, _dp, C.POINTER(RasterOpts), _fp], C.c_int),
    "hgs_backward": ([_vp, _vp, C.c_int, C.c_int, C.c_double], C.c_int),
    "hgs_zero_grads": ([_vp], C.c_int),
    "hgs_grads_download": ([_vp, C.POINTER(HostScene), C.c_int, _vp, _vp], C.c_int),
    "hgs_grads_device": ([_vp, C.POINTER(_fp), _i64p], C.c_int),
    "hgs_grads_packed": ([_vp, C.c_int, C.POINTER(_fp), _i64p], C.c_int),
    "hgs_loss_with_grad": ([_vp, _vp, C.c_int, C.c_int, C.c_double, _dp, _vp], C.c_int),
    "hgs_photometric_loss_with_grad": ([_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _vp], C.c_int),
    "hgs_adam_step": ([_vp, C.POINTER(Lrs), C.c_double, _i64p], C.c_int),
    "hgs_adam_state_download": ([_vp, C.POINTER(HostScene), C.POINTER(HostScene), C.c_int,
                                 C.POINTER(C.c_uint64)], C.c_int),
    "hgs_adam_state_upload": ([_vp, C.POINTER(HostScene), C.POINTER(HostScene), C.c_int, C.c_uint64], C.c_int),
    "hgs_stats_download": ([_vp, _dp, _u32p, _dp, _u32p], C.c_int),
    "hgs_sweep_convert": ([_vp, _i64p, C.POINTER(ConversionReport)], C.c_int),
    "hgs_train_step": ([_vp, C.c_int, C.POINTER(Camera_), _dp, C.POINTER(_fp), C.c_int, C.POINTER(TrainOpts),
                        C.c_int, _dp], C.c_int),
    "hgs_train_step_host": ([_vp, C.c_int, C.POINTER(Camera_), _dp, C.POINTER(_vp), C.c_int, C.c_int,
                             C.POINTER(TrainOpts), C.c_int, _dp], C.c_int),
    "hgs_densify_plan": ([_vp, C.POINTER(DensifyCfg), _vp, _vp, C.POINTER(DensifyReport)], C.c_int),
    "hgs_densify_apply": ([_vp, _dp, _dp, C.c_double], C.c_int),
    "hgs_opacity_reset": ([_vp, C.c_double], C.c_int),
    "hgs_render_sweep": ([_vp, C.c_int, C.POINTER(Camera_), _dp, _dp, C.POINTER(RasterOpts), _fp, C.c_int,
                          C.POINTER(RenderStats)], C.c_int),
    "hgs_rng_create": ([C.c_uint64, C.POINTER(_vp)], C.c_int),
    "hgs_rng_destroy": ([_vp], None),
    "hgs_rng_raw": ([_vp], C.c_uint64),
    "hgs_rng_index": ([_vp, C.c_uint64, C.c_uint64], C.c_uint64),
    "hgs_rng_batch": ([_vp, C.c_uint64, C.c_int32, C.POINTER(C.c_uint64)], C.c_int),
    "hgs_densify_normals": ([_vp, _vp, C.c_int64, _vp, C.c_int64, _dp, _dp], C.c_int),
    "hgs_densify_and_prune": ([_vp, C.POINTER(DensifyCfg), _vp, C.POINTER(DensifyReport)], C.c_int),
    "hgs_comm_unique_id": ([C.POINTER(CommId)], C.c_int),
    "hgs_comm_init": ([_vp, C.c_int, C.c_int, C.POINTER(CommId)], C.c_int),
    "hgs_comm_init_all": ([C.POINTER(_vp), C.c_int], C.c_int),
    "hgs_comm_destroy": ([_vp], C.c_int),
    "hgs_comm_nccl_info": ([C.POINTER(C.c_int), C.c_char_p, C.c_int], C.c_int),
    "hgs_comm_size": ([_vp], C.c_int),
    "hgs_comm_rank": ([_vp], C.c_int),
    "hgs_allreduce_grads": ([_vp], C.c_int),
    "hgs_allreduce_f64": ([_vp, _dp, C.c_int], C.c_int),
    "hgs_param_checksum": ([_vp, C.POINTER(C.c_uint64)], C.c_int),
    "hgs_broadcast_params": ([_vp, C.c_int], C.c_int),
    "hgs_init_scene": ([_vp, _dp, _dp, C.c_int64, C.POINTER(InitCfg)], C.c_int),
    "hgs_ppm_info": ([C.c_char_p, _i32p, _i32p], C.c_int),
    "hgs_ppm_read": ([C.c_char_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32], C.c_int),
    "hgs_ppm_read_batch": ([C.POINTER(C.c_char_p), C.c_int32, C.POINTER(C.POINTER(C.c_uint8)), C.c_int32, C.c_int32,
                            C.c_int32], C.c_int),
    "hgs_ppm_write": ([C.c_char_p, _vp, C.c_int, C.c_int32, C.c_int32], C.c_int),
    "hgs_image_last_error": ([], C.c_char_p),
    "hgs_checkpoint_save": ([_vp, C.c_char_p, C.c_int], C.c_int),
    "hgs_checkpoint_load": ([_vp, C.c_char_p, C.POINTER(C.c_int)], C.c_int),
    "hgs_checkpoint_write": ([C.POINTER(HostScene), C.POINTER(HostState), C.c_char_p], C.c_int),
    "hgs_checkpoint_info": ([C.c_char_p, _i64p, _i64p, _i32p, C.POINTER(C.c_int)], C.c_int),
    "hgs_checkpoint_read": ([C.c_char_p, C.POINTER(HostScene), C.POINTER(HostState)], C.c_int),
    "hgs_io_last_error": ([], C.c_char_p),
    "hgs_image_metrics": ([_vp, _vp, C.c_int, C.c_int, _dp, _dp], C.c_int),
    "hgs_metrics": ([_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp], C.c_int),
    "hgs_density_map": ([_vp, C.POINTER(Camera_), C.c_double, C.c_int, C.c_double, _u32p], C.c_int),
    "hgs_train_step_async": ([_vp, C.c_int, C.POINTER(Camera_), _dp, C.POINTER(_vp), C.c_int, C.c_int, C.c_int,
                              C.POINTER(TrainOpts), C.c_int], C.c_int),
    "hgs_train_collect": ([_vp, _dp], C.c_int),
    "hgs_train_exchange_async": ([_vp, C.POINTER(TrainOpts)], C.c_int),
    "hgs_train_pending": ([_vp], C.c_int),
    "hgs_profile": ([_vp, C.c_int], C.c_int),
    "hgs_profile_read": ([_vp, _dp, C.POINTER(C.c_longlong), C.c_int], C.c_int),
    "hgs_launch_count": ([], C.c_longlong),
}

PHASES = ("preprocess", "depth_sort", "duplicate", "tile_sort", "raster_fwd", "loss", "raster_bwd",
          "gaussian_bwd", "adam", "sweep", "upload")

# symbols every build must export (checked by the CPU test suite)
EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libhgs_gpu.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name, None)
            if f is None:
                continue
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check_io(rc: int) -> None:
    """Status of the context-free file entry points (message: hgs_io_last_error)."""
    if rc != 0:
        raise _STATUS.get(rc, HgsError)(lib().hgs_io_last_error().decode())


def check(ctx, rc: int) -> None:
    if rc != 0:
        msg = lib().hgs_last_error(ctx).decode() if ctx else f"status {rc}"
        raise _STATUS.get(rc, HgsError)(msg)


def camera_struct(cam) -> Camera_:
    k = Camera_()
    k.fx, k.fy, k.cx, k.cy = cam.fx, cam.fy, cam.cx, cam.cy
    r = np.asarray(cam.rot, dtype=np.float64).reshape(9)
    t = np.asarray(cam.trans, dtype=np.float64).reshape(3)
    for i in range(9):
        k.rot[i] = r[i]
    for i in range(3):
        k.trans[i] = t[i]
    k.width, k.height, k.near_, k.far_ = int(cam.width), int(cam.height), cam.near, cam.far
    return k


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_vp)
