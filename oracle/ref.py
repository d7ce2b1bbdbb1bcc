"""ctypes wrapper of oracle/_ref/libhgs_ref.so -- the REFERENCE library itself
(/root/reference/proj/src compiled against oracle/ref_shim, see
oracle/Makefile target ``ref``) behind a C ABI in the oracle's struct types
(oracle/ref_capi.cpp).  TEST INFRASTRUCTURE ONLY: pins the oracle restatement
against the reference's own code (tests/test_oracle_vs_reference.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import oracle as O
from paper_2505_13215_b200.scene import Camera, HybridScene

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libhgs_ref.so")
REF_SRC = "/root/reference/proj"

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build() -> bool:
    """Compile oracle/_ref when the reference sources are present."""
    if not os.path.isdir(os.path.join(REF_SRC, "src")):
        return available()
    subprocess.check_call(["make", "-s", "-j", str(min(8, os.cpu_count() or 4)), "-C", _HERE, "ref", "CXX=g++"])
    return True


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.hgsr_last_error.restype = C.c_char_p
        L.hgsr_rasterize.argtypes = [C.POINTER(O._Scene), C.POINTER(O._Camera), C.c_double, O._dp, C.c_double,
                                     C.c_int, O._dp, O._u32p, O._dp, C.POINTER(O._Stats)]
        L.hgsr_project_scene.argtypes = [C.POINTER(O._Scene), C.POINTER(O._Camera), C.c_double, C.c_double,
                                         C.c_void_p, C.c_int64, O._i64p, C.POINTER(O._Stats)]
        L.hgsr_forward_backward.argtypes = [C.POINTER(O._Scene), C.POINTER(O._Camera), C.c_double, O._dp,
                                            C.c_double, O._dp, O._dp, C.POINTER(O._Grads)]
        L.hgsr_photometric_loss_with_grad.restype = C.c_double
        L.hgsr_photometric_loss_with_grad.argtypes = [O._dp, O._dp, C.c_int, C.c_int, C.c_double, O._dp]
        L.hgsr_sweep_convert.argtypes = [C.POINTER(O._Scene), C.POINTER(O._Scene), O._i64p, C.POINTER(O._Conv)]
        L.hgsr_optimizer_step_fresh.argtypes = [C.POINTER(O._Scene), C.POINTER(O._Grads), C.POINTER(O._Lrs),
                                                C.c_double, C.c_int, C.POINTER(O._Scene), O._i64p]
        L.hgsr_set_quat_ctor.argtypes = [C.c_int]
        L.hgsr_save_checkpoint.argtypes = [C.POINTER(O._Scene), C.c_double, C.c_void_p, C.c_char_p]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise O._ERRS.get(rc, O.OracleError)(lib().hgsr_last_error().decode())


def rasterize(scene: HybridScene, cam: Camera, t: float, background=(0.0, 0.0, 0.0), num_threads: int = 1,
              weight_cutoff: float = 0.05, count_map: bool = False, transmittance_map: bool = False) -> dict:
    """hgs::rasterize (raster.hpp:79-80)."""
    st = O._scene_struct(scene)
    rgb = np.zeros((cam.height, cam.width, 3))
    counts = np.zeros((cam.height, cam.width), dtype=np.uint32) if count_map else None
    trans = np.zeros((cam.height, cam.width)) if transmittance_map else None
    stats = O._Stats()
    _check(lib().hgsr_rasterize(C.byref(st), C.byref(O._cam_struct(cam)), t, O._p(O._arr(background, 3)),
                                weight_cutoff, num_threads, O._p(rgb),
                                counts.ctypes.data_as(O._u32p) if counts is not None else None,
                                O._p(trans) if trans is not None else None, C.byref(stats)))
    return {"rgb": rgb, "counts": counts, "transmittance": trans, "stats": O._stats_dict(stats)}


def project_scene(scene: HybridScene, cam: Camera, t: float, weight_cutoff: float = 0.05):
    """hgs::project_scene (raster.hpp:74-76) as the oracle's splat records."""
    st = O._scene_struct(scene)
    n = C.c_int64()
    stats = O._Stats()
    cap = scene.n4 + scene.n3
    out = np.zeros(max(cap, 1), dtype=O.SPLAT_DTYPE)
    _check(lib().hgsr_project_scene(C.byref(st), C.byref(O._cam_struct(cam)), t, weight_cutoff,
                                    out.ctypes.data_as(C.c_void_p), cap, C.byref(n), C.byref(stats)))
    return out[: n.value].copy(), O._stats_dict(stats)


def forward_backward(scene: HybridScene, cam: Camera, t: float, background, loss_grad, weight_cutoff=0.05):
    """hgs::forward_train + hgs::backward (backward.hpp:68-74): image, grads."""
    st = O._scene_struct(scene)
    rgb = np.zeros((cam.height, cam.width, 3))
    if loss_grad is None:  # the taped forward only
        _check(lib().hgsr_forward_backward(C.byref(st), C.byref(O._cam_struct(cam)), t,
                                           O._p(O._arr(background, 3)), weight_cutoff, None, O._p(rgb), None))
        return rgb, None
    g = O.zero_grads(scene)
    lg = O._arr(loss_grad)
    _check(lib().hgsr_forward_backward(C.byref(st), C.byref(O._cam_struct(cam)), t, O._p(O._arr(background, 3)),
                                       weight_cutoff, O._p(lg), O._p(rgb), C.byref(O._grads_struct(g))))
    return rgb, g


def photometric_loss_with_grad(a, b, ssim_lambda=0.2):
    """hgs::photometric_loss_with_grad (loss.hpp:12-13)."""
    a, b = O._arr(a), O._arr(b)
    h, w = a.shape[:2]
    grad = np.zeros_like(a)
    loss = lib().hgsr_photometric_loss_with_grad(O._p(a), O._p(b), w, h, ssim_lambda, O._p(grad))
    return loss, grad


def sweep_convert(scene: HybridScene):
    """hgs::sweep_convert (scene.hpp:75): (converted scene, moved, report)."""
    n3, n4 = scene.n3, scene.n4
    out = O._empty_scene_like(scene, n4, n3 + n4)
    so = O._scene_struct(out)
    moved = np.zeros(max(n4, 1), dtype=np.int64)
    rep = O._Conv()
    _check(lib().hgsr_sweep_convert(C.byref(O._scene_struct(scene)), C.byref(so), moved.ctypes.data_as(O._i64p),
                                    C.byref(rep)))
    k4, k3 = int(so.n4), int(so.n3)
    for f in HybridScene.DYN_FIELDS:
        setattr(out, f, np.ascontiguousarray(getattr(out, f)[:k4]))
    for f in HybridScene.STA_FIELDS:
        setattr(out, f, np.ascontiguousarray(getattr(out, f)[:k3]))
    report = {"count": int(rep.count), "max_leakage": rep.max_leakage, "mean_leakage": rep.mean_leakage}
    return out, moved[: rep.count].copy(), report


def optimizer_steps(scene: HybridScene, grads: dict, n_steps: int = 1, lrs=None, mean_lr_scale: float = 1.0):
    """n x hgs::optimizer_step (train.hpp:68-69) from fresh Adam state with
    the same gradients: (updated scene, skipped_nonfinite)."""
    lrs = lrs or O.LearningRates()
    out = O._empty_scene_like(scene, scene.n4, scene.n3)
    so = O._scene_struct(out)
    sk = C.c_int64()
    _check(lib().hgsr_optimizer_step_fresh(C.byref(O._scene_struct(scene)), C.byref(O._grads_struct(grads)),
                                           C.byref(O._lrs_struct(lrs)), mean_lr_scale, n_steps, C.byref(so),
                                           C.byref(sk)))
    return out, int(sk.value)


def save_checkpoint(scene: HybridScene, path: str, state=None) -> None:
    """hgs::save_checkpoint (data_io.hpp:91-92); ``state``: an
    oracle.AdamState-like object (m, v, grad_norm*, count*, step,
    skipped_nonfinite) or None."""
    st = None
    if state is not None:
        st = O._State()
        st.m = O._scene_struct(state.m)
        st.v = O._scene_struct(state.v)
        keep = [np.ascontiguousarray(state.grad_norm4, np.float64), np.ascontiguousarray(state.grad_norm3, np.float64),
                np.ascontiguousarray(state.count4, np.uint32), np.ascontiguousarray(state.count3, np.uint32)]
        st.grad_norm4, st.grad_norm3 = O._p(keep[0]), O._p(keep[1])
        st.count4, st.count3 = keep[2].ctypes.data_as(O._u32p), keep[3].ctypes.data_as(O._u32p)
        st.step, st.skipped_nonfinite = int(state.step), int(state.skipped_nonfinite)
        st._keep = (state, keep)  # noqa: SLF001
    _check(lib().hgsr_save_checkpoint(C.byref(O._scene_struct(scene)), float(scene.duration_seconds),
                                      C.byref(st) if st is not None else None, path.encode()))
