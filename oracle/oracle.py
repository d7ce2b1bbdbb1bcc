"""ctypes wrapper of oracle/_build/libhgs_oracle.so (TEST INFRASTRUCTURE ONLY).

Mirrors the reference's ``hybridgs._core`` surface (python/bindings.cpp:35-236)
closely enough that parity tests read like the reference's own tests, but every
call here runs the CPU FP64 restatement, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2505_13215_b200.scene import Camera, HybridScene, sh_coeff_count

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libhgs_oracle.so")

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)


class _Scene(C.Structure):
    _fields_ = [("n4", C.c_int64), ("n3", C.c_int64), ("sh_degree", C.c_int32),
                ("tau", C.c_double), ("extent", C.c_double)] + [
        (n, _dp) for n in ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4",
                           "mean3", "quat3", "log_s3", "op3", "sh3")]


class _Grads(C.Structure):
    _fields_ = [(n, _dp) for n in ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4",
                                   "screen_norm4", "mean3", "quat3", "log_s3", "op3", "sh3",
                                   "screen_norm3")]


class _Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("rot", C.c_double * 9), ("trans", C.c_double * 3), ("width", C.c_int32),
                ("height", C.c_int32), ("near_", C.c_double), ("far_", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("culled_depth", "culled_offscreen", "culled_degenerate",
                                         "culled_temporal", "degenerate_temporal", "projected")]


class _Splat(C.Structure):
    _fields_ = [("sx", C.c_double), ("sy", C.c_double), ("conic", C.c_double * 4),
                ("depth", C.c_double), ("rgb", C.c_double * 3), ("alpha", C.c_double),
                ("radius", C.c_int32), ("pool", C.c_int32), ("index", C.c_int32),
                ("gid", C.c_int32), ("x0", C.c_int32), ("x1", C.c_int32), ("y0", C.c_int32),
                ("y1", C.c_int32), ("depth_bits", C.c_uint32), ("pad_", C.c_int32)]


SPLAT_DTYPE = np.dtype([("sx", "f8"), ("sy", "f8"), ("conic", "f8", (4,)), ("depth", "f8"),
                        ("rgb", "f8", (3,)), ("alpha", "f8"), ("radius", "i4"), ("pool", "i4"),
                        ("index", "i4"), ("gid", "i4"), ("x0", "i4"), ("x1", "i4"), ("y0", "i4"),
                        ("y1", "i4"), ("depth_bits", "u4"), ("pad_", "i4")])
assert SPLAT_DTYPE.itemsize == C.sizeof(_Splat)


class _State(C.Structure):
    _fields_ = [("m", _Scene), ("v", _Scene), ("grad_norm4", _dp), ("grad_norm3", _dp),
                ("count4", _u32p), ("count3", _u32p), ("step", C.c_uint64),
                ("skipped_nonfinite", C.c_uint64)]


class _Lrs(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mean", "mean_final_ratio", "mean_t", "quat", "scales",
                                          "opacity", "sh")]


class _DensifyCfg(C.Structure):
    _fields_ = [("grad_threshold", C.c_double), ("opacity_prune_eps", C.c_double),
                ("clone_size_frac", C.c_double), ("split_factor", C.c_double), ("max_gaussians", C.c_int64)]


class _DensifyRep(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("cloned3", "split3", "pruned3", "cloned4", "split4", "pruned4")]


class _Conv(C.Structure):
    _fields_ = [("count", C.c_int64), ("max_leakage", C.c_double), ("mean_leakage", C.c_double)]


class OracleError(RuntimeError):
    pass


class DegenerateTemporalError(OracleError):
    pass


class DegenerateRotationError(OracleError):
    pass


class NumericAbort(OracleError):
    pass


_ERRS = {1: ValueError, 2: DegenerateTemporalError, 3: DegenerateRotationError, 4: NumericAbort}


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (g++ -O3 -ffp-contract=off)."""
    src = os.path.join(_HERE, "hgs_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "CXX=g++"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.hgso_last_error.restype = C.c_char_p
        L.hgso_rng_new.restype = C.c_void_p
        L.hgso_rng_new.argtypes = [C.c_uint64]
        L.hgso_rng_free.argtypes = [C.c_void_p]
        for f in ("hgso_rng_uniform", "hgso_rng_normal"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [C.c_void_p]
        L.hgso_rng_index.restype = C.c_uint64
        L.hgso_rng_index.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.hgso_rng_raw.restype = C.c_uint64
        L.hgso_rng_raw.argtypes = [C.c_void_p]
        L.hgso_rng_normal_seq.argtypes = [C.c_void_p, C.c_int64, _dp]
        L.hgso_init_scene.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.POINTER(_Scene), _dp]
        L.hgso_density_map.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double, C.c_int, C.c_double,
                                       _u32p]
        L.hgso_densify_and_prune.argtypes = [C.POINTER(_Scene), C.POINTER(_State), C.POINTER(_Scene),
                                             C.POINTER(_State), C.POINTER(_DensifyCfg), C.c_void_p,
                                             C.POINTER(_DensifyRep)]
        L.hgso_random_scene.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(_Scene)]
        L.hgso_random_quat.argtypes = [C.c_void_p, _dp]
        L.hgso_random_camera.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(_Camera)]
        L.hgso_look_at.argtypes = [_dp, _dp, _dp, C.c_double, C.c_int, C.c_int, C.POINTER(_Camera)]
        L.hgso_exp.restype = C.c_double
        L.hgso_exp.argtypes = [C.c_double]
        for f in ("hgso_photometric_loss", "hgso_ssim", "hgso_psnr"):
            getattr(L, f).restype = C.c_double
        L.hgso_photometric_loss.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double]
        L.hgso_photometric_loss_with_grad.restype = C.c_double
        L.hgso_photometric_loss_with_grad.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, _dp]
        L.hgso_ssim.argtypes = [_dp, _dp, C.c_int, C.c_int]
        L.hgso_ssim_with_grad.restype = C.c_double
        L.hgso_ssim_with_grad.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp]
        L.hgso_psnr.argtypes = [_dp, _dp, C.c_int, C.c_int]
        L.hgso_tape_free.argtypes = [C.c_void_p]
        L.hgso_tape_contrib_total.restype = C.c_int64
        L.hgso_tape_contrib_total.argtypes = [C.c_void_p]
        L.hgso_forward_train.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double, _dp,
                                         C.c_double, C.c_int, _dp, C.POINTER(C.c_void_p)]
        L.hgso_forward_train_untiled.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double,
                                                 _dp, C.c_double, _dp, C.POINTER(C.c_void_p)]
        L.hgso_backward.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_void_p, _dp,
                                    C.POINTER(_Grads)]
        L.hgso_grads_add_scaled.argtypes = [C.POINTER(_Scene), C.POINTER(_Grads), C.POINTER(_Grads),
                                            C.c_double]
        L.hgso_project_scene.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double,
                                         C.c_double, C.c_void_p, C.c_int64, _i64p, C.POINTER(_Stats)]
        L.hgso_project_3d.argtypes = [_dp, _dp, C.POINTER(_Camera), C.c_void_p, C.POINTER(_Stats),
                                      C.POINTER(C.c_int)]
        L.hgso_sorted_instances.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double,
                                            C.c_double, _u32p, _u32p, C.c_int64, _i64p]
        L.hgso_rasterize.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double, _dp,
                                     C.c_double, C.c_int, _dp, _u32p, _dp, C.POINTER(_Stats)]
        L.hgso_reference_render.argtypes = [C.POINTER(_Scene), C.POINTER(_Camera), C.c_double, _dp,
                                            C.c_double, _dp, C.POINTER(_Stats)]
        L.hgso_optimizer_step.argtypes = [C.POINTER(_Scene), C.POINTER(_Grads), C.POINTER(_State),
                                          C.POINTER(_Lrs), C.c_double]
        L.hgso_accumulate_stats.argtypes = [C.POINTER(_Scene), C.POINTER(_State), C.POINTER(_Grads)]
        L.hgso_sweep_convert.argtypes = [C.POINTER(_Scene), C.POINTER(_State), _i64p, C.POINTER(_Conv)]
        L.hgso_is_static.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int)]
        L.hgso_convert_4d_to_3d.argtypes = [_dp, C.c_double, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp, _dp]
        L.hgso_condition_at_time.argtypes = [_dp, _dp, C.c_double, _dp, _dp, _dp]
        L.hgso_clamp_psd.argtypes = [_dp, C.c_double, _dp]
        L.hgso_extract_spatial_rot.argtypes = [_dp, _dp, _dp]
        L.hgso_sh_basis.argtypes = [_dp, C.c_int, _dp]
        L.hgso_sh_basis_grad.argtypes = [_dp, C.c_int, _dp]
        L.hgso_eval_sh.argtypes = [_dp, C.c_int, _dp, _dp]
        L.hgso_quat_to_rot3.argtypes = [_dp, _dp]
        L.hgso_rot3_to_quat.argtypes = [_dp, _dp]
        L.hgso_rot4_from_pair.argtypes = [_dp, _dp, _dp]
        L.hgso_build_cov4.argtypes = [_dp, _dp, _dp]
        L.hgso_build_cov3.argtypes = [_dp, _dp, _dp]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().hgso_last_error().decode()
        raise _ERRS.get(rc, OracleError)(msg)


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_dp)


def _arr(x, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _scene_struct(s: HybridScene) -> _Scene:
    st = _Scene()
    st.n4, st.n3, st.sh_degree, st.tau, st.extent = s.n4, s.n3, s.sh_degree, s.tau, s.extent
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        a = getattr(s, f)
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            a = np.ascontiguousarray(a, dtype=np.float64)
            setattr(s, f, a)
        setattr(st, f, _p(a))
    st._keep = s  # noqa: SLF001
    return st


def _cam_struct(c: Camera) -> _Camera:
    k = _Camera()
    k.fx, k.fy, k.cx, k.cy = c.fx, c.fy, c.cx, c.cy
    r = np.asarray(c.rot, dtype=np.float64).reshape(9)
    t = np.asarray(c.trans, dtype=np.float64).reshape(3)
    for i in range(9):
        k.rot[i] = r[i]
    for i in range(3):
        k.trans[i] = t[i]
    k.width, k.height, k.near_, k.far_ = c.width, c.height, c.near, c.far
    return k


def _camera_from(k: _Camera) -> Camera:
    return Camera(fx=k.fx, fy=k.fy, cx=k.cx, cy=k.cy, rot=np.array(list(k.rot)).reshape(3, 3),
                  trans=np.array(list(k.trans)), width=k.width, height=k.height, near=k.near_,
                  far=k.far_)


def _stats_dict(s: _Stats) -> dict:
    return {n: int(getattr(s, n)) for n, _ in _Stats._fields_}


# --------------------------------------------------------------- fixtures
class Rng:
    """std::mt19937_64 + libstdc++ distributions (tests/oracles.hpp)."""

    def __init__(self, seed: int):
        self._h = lib().hgso_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().hgso_rng_free(self._h)
            self._h = None

    def uniform(self) -> float:
        return lib().hgso_rng_uniform(self._h)

    def normal(self) -> float:
        return lib().hgso_rng_normal(self._h)

    def index(self, lo: int, hi: int) -> int:
        """std::uniform_int_distribution<size_t>(lo, hi) (train.cpp:392)."""
        return lib().hgso_rng_index(self._h, lo, hi)

    def raw(self) -> int:
        return lib().hgso_rng_raw(self._h)

    def normal_seq(self, n: int) -> np.ndarray:
        """n draws from ONE std::normal_distribution object."""
        out = np.zeros(max(n, 1))
        lib().hgso_rng_normal_seq(self._h, n, _p(out))
        return out[:n]

    def random_quat(self) -> np.ndarray:
        q = np.zeros(4)
        lib().hgso_random_quat(self._h, _p(q))
        return q

    def random_scene(self, n_static: int, n_dynamic: int, sh_degree: int = 1) -> HybridScene:
        K = sh_coeff_count(sh_degree)
        s = HybridScene(sh_degree=sh_degree, extent=2.0)
        s.mean_x, s.mean_t = np.zeros((n_dynamic, 3)), np.zeros(n_dynamic)
        s.ql, s.qr, s.log_s4 = np.zeros((n_dynamic, 4)), np.zeros((n_dynamic, 4)), np.zeros((n_dynamic, 4))
        s.op4, s.sh4 = np.zeros(n_dynamic), np.zeros((n_dynamic, K, 3))
        s.mean3, s.quat3, s.log_s3 = np.zeros((n_static, 3)), np.zeros((n_static, 4)), np.zeros((n_static, 3))
        s.op3, s.sh3 = np.zeros(n_static), np.zeros((n_static, K, 3))
        st = _scene_struct(s)
        lib().hgso_random_scene(self._h, n_static, n_dynamic, sh_degree, C.byref(st))
        s.extent = st.extent
        return s

    def random_camera(self, width: int = 64, height: int = 64) -> Camera:
        k = _Camera()
        _check(lib().hgso_random_camera(self._h, width, height, C.byref(k)))
        return _camera_from(k)


def look_at(eye, target, up, focal, width, height) -> Camera:
    k = _Camera()
    _check(lib().hgso_look_at(_p(_arr(eye, 3)), _p(_arr(target, 3)), _p(_arr(up, 3)), focal,
                              width, height, C.byref(k)))
    return _camera_from(k)


# --------------------------------------------------------------- math
def quat_to_rot3(q) -> np.ndarray:
    r = np.zeros(9)
    _check(lib().hgso_quat_to_rot3(_p(_arr(q, 4)), _p(r)))
    return r.reshape(3, 3)


def rot3_to_quat(r) -> np.ndarray:
    q = np.zeros(4)
    _check(lib().hgso_rot3_to_quat(_p(_arr(r, 9)), _p(q)))
    return q


def rot4_from_pair(ql, qr) -> np.ndarray:
    r = np.zeros(16)
    lib().hgso_rot4_from_pair(_p(_arr(ql, 4)), _p(_arr(qr, 4)), _p(r))
    return r.reshape(4, 4)


def build_cov4(rot4, log_s) -> np.ndarray:
    c = np.zeros(16)
    lib().hgso_build_cov4(_p(_arr(rot4, 16)), _p(_arr(log_s, 4)), _p(c))
    return c.reshape(4, 4)


def build_cov3(rot3, log_s) -> np.ndarray:
    c = np.zeros(9)
    lib().hgso_build_cov3(_p(_arr(rot3, 9)), _p(_arr(log_s, 3)), _p(c))
    return c.reshape(3, 3)


def condition_at_time(mean4, cov4, t):
    m3, c3, w = np.zeros(3), np.zeros(9), C.c_double()
    _check(lib().hgso_condition_at_time(_p(_arr(mean4, 4)), _p(_arr(cov4, 16)), t, _p(m3), _p(c3),
                                        C.byref(w)))
    return m3, c3.reshape(3, 3), w.value


def clamp_psd(m, eps=1e-12) -> np.ndarray:
    out = np.zeros(9)
    _check(lib().hgso_clamp_psd(_p(_arr(m, 9)), eps, _p(out)))
    return out.reshape(3, 3)


def extract_spatial_rot(rot4):
    r3, leak = np.zeros(9), C.c_double()
    _check(lib().hgso_extract_spatial_rot(_p(_arr(rot4, 16)), _p(r3), C.byref(leak)))
    return r3.reshape(3, 3), leak.value


def sh_basis(direction, degree) -> np.ndarray:
    out = np.zeros(16)
    lib().hgso_sh_basis(_p(_arr(direction, 3)), degree, _p(out))
    return out[: sh_coeff_count(degree)]


def sh_basis_grad(direction, degree) -> np.ndarray:
    out = np.zeros(48)
    lib().hgso_sh_basis_grad(_p(_arr(direction, 3)), degree, _p(out))
    return out.reshape(16, 3)[: sh_coeff_count(degree)]


def eval_sh(coeffs, degree, direction) -> np.ndarray:
    rgb = np.zeros(3)
    _check(lib().hgso_eval_sh(_p(_arr(coeffs).reshape(-1)), degree, _p(_arr(direction, 3)), _p(rgb)))
    return rgb


def cexp(x: float) -> float:
    """The host libm exp the oracle uses."""
    return lib().hgso_exp(x)


def is_static(log_st: float, tau: float) -> bool:
    out = C.c_int()
    _check(lib().hgso_is_static(log_st, tau, C.byref(out)))
    return bool(out.value)


def convert_4d_to_3d(mean_x, mean_t, ql, qr, log_s4, op):
    m3, q3, ls3, o3 = np.zeros(3), np.zeros(4), np.zeros(3), np.zeros(1)
    _check(lib().hgso_convert_4d_to_3d(_p(_arr(mean_x, 3)), mean_t, _p(_arr(ql, 4)), _p(_arr(qr, 4)),
                                       _p(_arr(log_s4, 4)), op, _p(m3), _p(q3), _p(ls3), _p(o3)))
    return m3, q3, ls3, float(o3[0])


# --------------------------------------------------------------- renderer
def project_scene(scene: HybridScene, cam: Camera, t: float, weight_cutoff: float = 0.05):
    st = _scene_struct(scene)
    out = np.zeros(scene.total(), dtype=SPLAT_DTYPE)
    n = C.c_int64()
    stats = _Stats()
    _check(lib().hgso_project_scene(C.byref(st), C.byref(_cam_struct(cam)), t, weight_cutoff,
                                    out.ctypes.data_as(C.c_void_p), len(out), C.byref(n),
                                    C.byref(stats)))
    return out[: n.value].copy(), _stats_dict(stats)


def project_3d(mean3, cov3, cam: Camera, stats: dict | None = None):
    """project_3d (raster.cpp:26-64); returns a splat record or None; updates ``stats``."""
    out = np.zeros(1, dtype=SPLAT_DTYPE)
    st = _Stats()
    if stats:
        for k, v in stats.items():
            setattr(st, k, v)
    ok = C.c_int()
    _check(lib().hgso_project_3d(_p(_arr(mean3, 3)), _p(_arr(cov3, 9)), C.byref(_cam_struct(cam)),
                                 out.ctypes.data_as(C.c_void_p), C.byref(st), C.byref(ok)))
    if stats is not None:
        stats.update(_stats_dict(st))
    return out[0] if ok.value else None


def sorted_instances(scene: HybridScene, cam: Camera, t: float, weight_cutoff: float = 0.05):
    """(tile_id, projected prim index) of every instance in reference sort order."""
    st = _scene_struct(scene)
    k = _cam_struct(cam)
    n = C.c_int64()
    _check(lib().hgso_sorted_instances(C.byref(st), C.byref(k), t, weight_cutoff, None, None, 0,
                                       C.byref(n)))
    tiles = np.zeros(n.value, dtype=np.uint32)
    prims = np.zeros(n.value, dtype=np.uint32)
    _check(lib().hgso_sorted_instances(C.byref(st), C.byref(k), t, weight_cutoff,
                                       tiles.ctypes.data_as(_u32p), prims.ctypes.data_as(_u32p),
                                       n.value, C.byref(n)))
    return tiles, prims


def rasterize(scene: HybridScene, cam: Camera, t: float, background=(0.0, 0.0, 0.0),
              num_threads: int = 1, weight_cutoff: float = 0.05, count_map: bool = False,
              transmittance_map: bool = False) -> dict:
    st = _scene_struct(scene)
    rgb = np.zeros((cam.height, cam.width, 3))
    counts = np.zeros((cam.height, cam.width), dtype=np.uint32) if count_map else None
    trans = np.zeros((cam.height, cam.width)) if transmittance_map else None
    stats = _Stats()
    _check(lib().hgso_rasterize(C.byref(st), C.byref(_cam_struct(cam)), t, _p(_arr(background, 3)),
                                weight_cutoff, num_threads, _p(rgb),
                                counts.ctypes.data_as(_u32p) if counts is not None else None,
                                _p(trans) if trans is not None else None, C.byref(stats)))
    return {"rgb": rgb, "counts": counts, "transmittance": trans, "stats": _stats_dict(stats)}


def reference_render(scene: HybridScene, cam: Camera, t: float, background=(0.0, 0.0, 0.0),
                     weight_cutoff: float = 0.05) -> np.ndarray:
    st = _scene_struct(scene)
    rgb = np.zeros((cam.height, cam.width, 3))
    _check(lib().hgso_reference_render(C.byref(st), C.byref(_cam_struct(cam)), t,
                                       _p(_arr(background, 3)), weight_cutoff, _p(rgb), None))
    return rgb


# --------------------------------------------------------------- training
class Tape:
    def __init__(self, handle):
        self._h = handle

    def contrib_total(self) -> int:
        return int(lib().hgso_tape_contrib_total(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().hgso_tape_free(self._h)
            self._h = None


GRAD_FIELDS = ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4", "screen_norm4",
               "mean3", "quat3", "log_s3", "op3", "sh3", "screen_norm3")


def zero_grads(scene: HybridScene) -> dict:
    g = {f: np.zeros_like(getattr(scene, f)) for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS}
    g["screen_norm4"] = np.zeros(scene.n4)
    g["screen_norm3"] = np.zeros(scene.n3)
    return g


def _grads_struct(g: dict) -> _Grads:
    st = _Grads()
    for f in GRAD_FIELDS:
        setattr(st, f, _p(g[f]))
    st._keep = g  # noqa: SLF001
    return st


def forward_train(scene: HybridScene, cam: Camera, t: float, background=(0.0, 0.0, 0.0),
                  weight_cutoff: float = 0.05, num_threads: int = 1, untiled: bool = False):
    st = _scene_struct(scene)
    rgb = np.zeros((cam.height, cam.width, 3))
    h = C.c_void_p()
    if untiled:
        _check(lib().hgso_forward_train_untiled(C.byref(st), C.byref(_cam_struct(cam)), t,
                                                _p(_arr(background, 3)), weight_cutoff, _p(rgb),
                                                C.byref(h)))
    else:
        _check(lib().hgso_forward_train(C.byref(st), C.byref(_cam_struct(cam)), t,
                                        _p(_arr(background, 3)), weight_cutoff, num_threads, _p(rgb),
                                        C.byref(h)))
    return rgb, Tape(h.value)


def backward(scene: HybridScene, cam: Camera, tape: Tape, loss_grad: np.ndarray,
             grads: dict | None = None) -> dict:
    """Accumulates into ``grads`` (zero-initialised when None), backward.hpp:71-74."""
    if grads is None:
        grads = zero_grads(scene)
    st = _scene_struct(scene)
    lg = _arr(loss_grad)
    _check(lib().hgso_backward(C.byref(st), C.byref(_cam_struct(cam)), tape._h, _p(lg),
                               C.byref(_grads_struct(grads))))
    return grads


def grads_add_scaled(scene: HybridScene, acc: dict, other: dict, scale: float) -> None:
    lib().hgso_grads_add_scaled(C.byref(_scene_struct(scene)), C.byref(_grads_struct(acc)),
                                C.byref(_grads_struct(other)), scale)


def photometric_loss(a, b, ssim_lambda=0.2) -> float:
    a, b = _arr(a), _arr(b)
    if a.shape != b.shape:
        raise ValueError("photometric_loss: image dimensions differ")
    return lib().hgso_photometric_loss(_p(a), _p(b), a.shape[1], a.shape[0], ssim_lambda)


def photometric_loss_with_grad(a, b, ssim_lambda=0.2):
    a, b = _arr(a), _arr(b)
    if a.shape != b.shape:
        raise ValueError("photometric_loss: image dimensions differ")
    g = np.zeros_like(a)
    loss = lib().hgso_photometric_loss_with_grad(_p(a), _p(b), a.shape[1], a.shape[0], ssim_lambda, _p(g))
    return loss, g


def ssim(a, b) -> float:
    a, b = _arr(a), _arr(b)
    if a.shape != b.shape:
        raise ValueError("metrics: image dimensions differ")
    if a.shape[0] < 11 or a.shape[1] < 11:
        raise ValueError("ssim: images smaller than the 11x11 window")
    return lib().hgso_ssim(_p(a), _p(b), a.shape[1], a.shape[0])


def ssim_with_grad(a, b):
    a, b = _arr(a), _arr(b)
    g = np.zeros_like(a)
    s = lib().hgso_ssim_with_grad(_p(a), _p(b), a.shape[1], a.shape[0], _p(g))
    return s, g


def psnr(a, b) -> float:
    a, b = _arr(a), _arr(b)
    if a.shape != b.shape:
        raise ValueError("metrics: image dimensions differ")
    return lib().hgso_psnr(_p(a), _p(b), a.shape[1], a.shape[0])


@dataclass
class LearningRates:  # train.hpp:13-21
    mean: float = 1.6e-4
    mean_final_ratio: float = 0.01
    mean_t: float = 1.6e-4
    quat: float = 1e-3
    scales: float = 5e-3
    opacity: float = 5e-2
    sh: float = 2.5e-3


class AdamState:
    """GradAccum (optim.hpp:32-41) with m/v laid out like the scene."""

    def __init__(self, scene: HybridScene):
        self.m = scene.copy()
        self.v = scene.copy()
        for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
            getattr(self.m, f)[...] = 0.0
            getattr(self.v, f)[...] = 0.0
        self.grad_norm4 = np.zeros(scene.n4)
        self.grad_norm3 = np.zeros(scene.n3)
        self.count4 = np.zeros(scene.n4, dtype=np.uint32)
        self.count3 = np.zeros(scene.n3, dtype=np.uint32)
        self.step = 0
        self.skipped_nonfinite = 0

    def _struct(self) -> _State:
        s = _State()
        s.m = _scene_struct(self.m)
        s.v = _scene_struct(self.v)
        s.grad_norm4, s.grad_norm3 = _p(self.grad_norm4), _p(self.grad_norm3)
        s.count4 = self.count4.ctypes.data_as(_u32p)
        s.count3 = self.count3.ctypes.data_as(_u32p)
        s.step, s.skipped_nonfinite = self.step, self.skipped_nonfinite
        s._keep = self  # noqa: SLF001
        return s


def _lrs_struct(l: LearningRates) -> _Lrs:
    k = _Lrs()
    for n, _ in _Lrs._fields_:
        setattr(k, n, getattr(l, n))
    return k


def optimizer_step(scene: HybridScene, grads: dict, state: AdamState, lrs: LearningRates | None = None,
                   mean_lr_scale: float = 1.0) -> None:
    lrs = lrs or LearningRates()
    st = state._struct()
    _check(lib().hgso_optimizer_step(C.byref(_scene_struct(scene)), C.byref(_grads_struct(grads)),
                                     C.byref(st), C.byref(_lrs_struct(lrs)), mean_lr_scale))
    state.step, state.skipped_nonfinite = st.step, st.skipped_nonfinite


def accumulate_stats(scene: HybridScene, state: AdamState, grads: dict) -> None:
    st = state._struct()
    lib().hgso_accumulate_stats(C.byref(_scene_struct(scene)), C.byref(st), C.byref(_grads_struct(grads)))


def _grow_statics(s: HybridScene, extra: int) -> None:
    for f in HybridScene.STA_FIELDS:
        a = getattr(s, f)
        pad = np.zeros((extra,) + a.shape[1:], dtype=a.dtype)
        setattr(s, f, np.ascontiguousarray(np.concatenate([a, pad], axis=0)))


def sweep_convert(scene: HybridScene, state: AdamState | None = None):
    """sweep_convert (scene.cpp:43-71) + remap_after_sweep (train.cpp:305-362).

    Mutates ``scene``/``state`` (arrays are replaced by resized copies) and
    returns (moved indices, report dict).
    """
    n3, n4 = scene.n3, scene.n4
    _grow_statics(scene, n4)
    if state is not None:
        _grow_statics(state.m, n4)
        _grow_statics(state.v, n4)
        state.grad_norm3 = np.zeros(n3 + n4)
        state.count3 = np.zeros(n3 + n4, dtype=np.uint32)
    st_scene = _scene_struct(scene)
    st_scene.n3 = n3  # logical size before the sweep
    moved = np.zeros(max(n4, 1), dtype=np.int64)
    rep = _Conv()
    st_state = state._struct() if state is not None else None
    if st_state is not None:
        st_state.m.n3 = n3
        st_state.v.n3 = n3
    _check(lib().hgso_sweep_convert(C.byref(st_scene), C.byref(st_state) if st_state else None,
                                    moved.ctypes.data_as(_i64p), C.byref(rep)))
    new_n3, new_n4 = int(st_scene.n3), int(st_scene.n4)
    for f in HybridScene.STA_FIELDS:
        setattr(scene, f, np.ascontiguousarray(getattr(scene, f)[:new_n3]))
    for f in HybridScene.DYN_FIELDS:
        setattr(scene, f, np.ascontiguousarray(getattr(scene, f)[:new_n4]))
    if state is not None:
        for b in (state.m, state.v):
            for f in HybridScene.STA_FIELDS:
                setattr(b, f, np.ascontiguousarray(getattr(b, f)[:new_n3]))
            for f in HybridScene.DYN_FIELDS:
                setattr(b, f, np.ascontiguousarray(getattr(b, f)[:new_n4]))
        state.grad_norm3 = np.zeros(new_n3)
        state.count3 = np.zeros(new_n3, dtype=np.uint32)
        state.grad_norm4 = np.zeros(new_n4)
        state.count4 = np.zeros(new_n4, dtype=np.uint32)
    report = {"count": int(rep.count), "max_leakage": rep.max_leakage, "mean_leakage": rep.mean_leakage}
    return moved[: rep.count].copy(), report


def densify_and_prune(scene: HybridScene, state: AdamState, rng: Rng, grad_threshold=0.02, opacity_prune_eps=0.005,
                      clone_size_frac=0.01, split_factor=1.6, max_gaussians=20000):
    """densify_and_prune (train.cpp:182-299): returns (new scene, new state,
    report dict); ``rng`` is advanced exactly like the reference's."""
    cap4, cap3 = 2 * scene.n4, 2 * scene.n3
    out = _empty_scene_like(scene, cap4, cap3)
    ost = AdamState(out)
    st_in, st_out = state._struct(), ost._struct()
    so = _scene_struct(out)
    cfg = _DensifyCfg(grad_threshold, opacity_prune_eps, clone_size_frac, split_factor, max_gaussians)
    rep = _DensifyRep()
    _check(lib().hgso_densify_and_prune(C.byref(_scene_struct(scene)), C.byref(st_in), C.byref(so), C.byref(st_out),
                                        C.byref(cfg), rng._h, C.byref(rep)))
    n4, n3 = int(so.n4), int(so.n3)
    for obj in (out, ost.m, ost.v):
        for f in HybridScene.DYN_FIELDS:
            setattr(obj, f, np.ascontiguousarray(getattr(obj, f)[:n4]))
        for f in HybridScene.STA_FIELDS:
            setattr(obj, f, np.ascontiguousarray(getattr(obj, f)[:n3]))
    ost.grad_norm4, ost.count4 = np.zeros(n4), np.zeros(n4, dtype=np.uint32)
    ost.grad_norm3, ost.count3 = np.zeros(n3), np.zeros(n3, dtype=np.uint32)
    ost.step, ost.skipped_nonfinite = state.step, state.skipped_nonfinite
    return out, ost, {n: int(getattr(rep, n)) for n, _ in _DensifyRep._fields_}


def density_map(scene: HybridScene, cam: Camera, t: float, dynamics_only: bool = False,
                weight_cutoff: float = 0.05) -> np.ndarray:
    """raster.cpp:268-287: (h, w) uint32 box-coverage counts."""
    out = np.zeros((cam.height, cam.width), dtype=np.uint32)
    _check(lib().hgso_density_map(C.byref(_scene_struct(scene)), C.byref(_cam_struct(cam)), t,
                                  1 if dynamics_only else 0, weight_cutoff, out.ctypes.data_as(_u32p)))
    return out


def init_scene(positions, rgb, sh_degree=1, tau=0.5, duration_seconds=1.0, init_temporal_scale=0.1,
               init_opacity=0.1) -> HybridScene:
    """data_io.cpp:189-238 (InitConfig defaults, data_io.hpp:43-49)."""
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    col = np.ascontiguousarray(rgb, dtype=np.float64).reshape(-1, 3)
    n = pos.shape[0]
    out = _empty_scene_like(HybridScene(sh_degree=sh_degree), n, 0)
    st = _scene_struct(out)
    dur = C.c_double()
    _check(lib().hgso_init_scene(_p(pos), _p(col), n, sh_degree, tau, duration_seconds, init_temporal_scale,
                                 init_opacity, C.byref(st), C.byref(dur)))
    out.tau, out.extent, out.duration_seconds = st.tau, st.extent, dur.value
    return out


def _empty_scene_like(scene: HybridScene, n4: int, n3: int) -> HybridScene:
    K = sh_coeff_count(scene.sh_degree)
    s = HybridScene(sh_degree=scene.sh_degree, tau=scene.tau, extent=scene.extent)
    s.mean_x, s.mean_t = np.zeros((n4, 3)), np.zeros(n4)
    s.ql, s.qr, s.log_s4 = np.zeros((n4, 4)), np.zeros((n4, 4)), np.zeros((n4, 4))
    s.op4, s.sh4 = np.zeros(n4), np.zeros((n4, K, 3))
    s.mean3, s.quat3, s.log_s3 = np.zeros((n3, 3)), np.zeros((n3, 4)), np.zeros((n3, 3))
    s.op3, s.sh3 = np.zeros(n3), np.zeros((n3, K, 3))
    return s


def hardware_threads() -> int:
    return int(lib().hgso_hardware_threads())


def train_step(scene: HybridScene, state: AdamState, cams, times, gts, background=(0.0, 0.0, 0.0),
               weight_cutoff: float = 0.05, ssim_lambda: float = 0.2, lrs: LearningRates | None = None,
               mean_lr_scale: float = 1.0, num_threads: int = 1, tile_threads: int = 1) -> float:
    """One iteration of train_scene's loop body (train.cpp:402-450); mutates
    scene and state, returns the mean batch loss."""
    L = lib()
    if not hasattr(L, "_ts_bound"):
        L.hgso_train_step.argtypes = [C.POINTER(_Scene), C.POINTER(_State), C.POINTER(_Camera), _dp,
                                      C.POINTER(_dp), C.c_int, _dp, C.c_double, C.c_double, C.POINTER(_Lrs),
                                      C.c_double, C.c_int, C.c_int, _dp]
        L._ts_bound = True
    n = len(cams)
    karr = (_Camera * n)(*[_cam_struct(c) for c in cams])
    tarr = (C.c_double * n)(*times)
    g = [_arr(x) for x in gts]
    garr = (_dp * n)(*[_p(x) for x in g])
    st = state._struct()
    loss = C.c_double()
    _check(L.hgso_train_step(C.byref(_scene_struct(scene)), C.byref(st), karr, tarr, garr, n,
                             _p(_arr(background, 3)), weight_cutoff, ssim_lambda,
                             C.byref(_lrs_struct(lrs or LearningRates())), mean_lr_scale, num_threads,
                             tile_threads, C.byref(loss)))
    state.step, state.skipped_nonfinite = st.step, st.skipped_nonfinite
    return loss.value
