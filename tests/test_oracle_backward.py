"""Pins the oracle's analytic gradients (test_backward.cpp:116-246) with
central finite differences of L = sum(W * rasterize(...))."""
import math

import numpy as np
import pytest

import oracle as O


def logit(p):
    return math.log(p / (1.0 - p))


class Setup:
    """test_backward.cpp:26-44 (same rng draw order)."""

    def __init__(self, seed):
        rng = O.Rng(seed)
        self.scene = rng.random_scene(3, 3)
        for i in range(self.scene.n3):
            self.scene.op3[i] = logit(0.3 + 0.5 * rng.uniform())
        for i in range(self.scene.n4):
            self.scene.op4[i] = logit(0.3 + 0.5 * rng.uniform())
            self.scene.log_s4[i, 3] = math.log(0.5 + 0.5 * rng.uniform())
            self.scene.mean_t[i] = 0.3 + 0.4 * rng.uniform()
        self.cam = rng.random_camera(32, 32)
        self.w = np.array([2.0 * rng.uniform() - 1.0 for _ in range(32 * 32 * 3)]).reshape(32, 32, 3)
        self.t = 0.45
        self.bg = (0.15, 0.2, 0.25)

    def loss(self):
        img = O.rasterize(self.scene, self.cam, self.t, self.bg)["rgb"]
        return float((self.w * img).sum())


def rel_err(a, b):  # test_backward.cpp:60-62
    return abs(a - b) / max(abs(a), abs(b), 1e-6)


def normalized(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3])
    v = v / n
    flip = v[0] < 0 or (v[0] == 0 and ((v[1] < 0) if v[1] != 0 else ((v[2] < 0) if v[2] != 0 else v[3] < 0)))
    return -v if flip else v


class Stats:
    def __init__(self):
        self.checked = self.skipped = self.failed = 0
        self.worst = 0.0


def check_param(su, analytic, setter, st):
    """test_backward.cpp:68-94"""
    def ev(d):
        setter(d)
        v = su.loss()
        setter(0.0)
        return v

    h = 1e-5
    fd1 = (ev(h) - ev(-h)) / (2 * h)
    if rel_err(analytic, fd1) < 1e-3:
        st.checked += 1
        return
    fd2 = (ev(0.25 * h) - ev(-0.25 * h)) / (0.5 * h)
    if rel_err(fd1, fd2) > 5e-4:
        st.skipped += 1
        return
    st.checked += 1
    e = rel_err(analytic, fd2)
    if e >= 1e-3:
        st.failed += 1
        st.worst = max(st.worst, e)


def analytic(su):
    img, tape = O.forward_train(su.scene, su.cam, su.t, su.bg)
    ref = O.rasterize(su.scene, su.cam, su.t, su.bg)["rgb"]
    assert (img == ref).all()
    return O.backward(su.scene, su.cam, tape, su.w)


def require_clean(st):  # test_backward.cpp:107-112
    assert st.checked > 0
    assert st.failed == 0, st.worst
    assert st.skipped * 10 <= st.checked


def _vec_setter(arr, idx):
    base = arr[idx]

    def f(d):
        arr[idx] = base + d
    return f


def _quat_setter(arr, i, c):
    q0 = arr[i].copy()

    def f(d):
        v = q0.copy()
        v[c] += d
        arr[i] = normalized(v) if d != 0.0 else q0
    return f


@pytest.mark.parametrize("seed", [61, 62, 63, 64])
def test_static_gradients_fd(seed):
    su = Setup(seed)
    g = analytic(su)
    sc = su.scene
    st = {k: Stats() for k in ("mean", "quat", "scales", "opacity", "sh")}
    for i in range(sc.n3):
        for c in range(3):
            check_param(su, g["mean3"][i, c], _vec_setter(sc.mean3, (i, c)), st["mean"])
        for c in range(4):
            check_param(su, g["quat3"][i, c], _quat_setter(sc.quat3, i, c), st["quat"])
        for c in range(3):
            check_param(su, g["log_s3"][i, c], _vec_setter(sc.log_s3, (i, c)), st["scales"])
        check_param(su, g["op3"][i], _vec_setter(sc.op3, i), st["opacity"])
        for k in range(sc.sh3.shape[1]):
            for c in range(3):
                check_param(su, g["sh3"][i, k, c], _vec_setter(sc.sh3, (i, k, c)), st["sh"])
    for v in st.values():
        require_clean(v)


@pytest.mark.parametrize("seed", [71, 72, 73, 74])
def test_dynamic_gradients_fd(seed):
    su = Setup(seed)
    g = analytic(su)
    sc = su.scene
    st = {k: Stats() for k in ("mean_x", "mean_t", "ql", "qr", "scales", "opacity", "sh")}
    for i in range(sc.n4):
        for c in range(3):
            check_param(su, g["mean_x"][i, c], _vec_setter(sc.mean_x, (i, c)), st["mean_x"])
        check_param(su, g["mean_t"][i], _vec_setter(sc.mean_t, i), st["mean_t"])
        for c in range(4):
            check_param(su, g["ql"][i, c], _quat_setter(sc.ql, i, c), st["ql"])
            check_param(su, g["qr"][i, c], _quat_setter(sc.qr, i, c), st["qr"])
        for c in range(4):
            check_param(su, g["log_s4"][i, c], _vec_setter(sc.log_s4, (i, c)), st["scales"])
        check_param(su, g["op4"][i], _vec_setter(sc.op4, i), st["opacity"])
        for k in range(sc.sh4.shape[1]):
            for c in range(3):
                check_param(su, g["sh4"][i, k, c], _vec_setter(sc.sh4, (i, k, c)), st["sh"])
    for v in st.values():
        require_clean(v)


def test_screen_norms_positive():
    """test_backward.cpp:214-229"""
    su = Setup(81)
    g = analytic(su)
    allv = np.concatenate([g["screen_norm3"], g["screen_norm4"]])
    assert np.isfinite(allv).all() and (allv >= 0).all() and (allv > 0).any()


def test_add_scaled():
    """test_backward.cpp:231-246"""
    su = Setup(82)
    a = analytic(su)
    acc = O.zero_grads(su.scene)
    O.grads_add_scaled(su.scene, acc, a, 0.25)
    O.grads_add_scaled(su.scene, acc, a, 0.75)
    assert np.abs(acc["mean3"] - a["mean3"]).max() < 1e-12
    assert np.abs(acc["log_s4"] - a["log_s4"]).max() < 1e-12
    assert np.allclose(acc["op3"], a["op3"], rtol=1e-12)
