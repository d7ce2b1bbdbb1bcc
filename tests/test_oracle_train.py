"""Pins the oracle's loss/metrics, Adam and 4D->3D conversion against the
reference's test_metrics.cpp, test_train.cpp and test_scene.cpp."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2505_13215_b200.scene import HybridScene

C0 = 0.28209479177387814


def logit(p):
    return math.log(p / (1.0 - p))


# ------------------------------------------------------------------ metrics
def ssim_ref(a, b):
    """test_metrics.cpp:35-70, an independent scalar SSIM (vectorised)."""
    ax = np.arange(11) - 5
    k = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2 * 1.5 * 1.5))
    k /= k.sum()
    H, W, _ = a.shape
    from numpy.lib.stride_tricks import sliding_window_view as swv
    total, count = 0.0, 0
    for ch in range(3):
        A = swv(a[:, :, ch], (11, 11))
        B = swv(b[:, :, ch], (11, 11))
        mu_a = (A * k).sum((-1, -2))
        mu_b = (B * k).sum((-1, -2))
        aa = (A * A * k).sum((-1, -2))
        bb = (B * B * k).sum((-1, -2))
        ab = (A * B * k).sum((-1, -2))
        va, vb, cv = aa - mu_a ** 2, bb - mu_b ** 2, ab - mu_a * mu_b
        s = ((2 * mu_a * mu_b + 1e-4) * (2 * cv + 9e-4)) / ((mu_a ** 2 + mu_b ** 2 + 1e-4) * (va + vb + 9e-4))
        total += s.sum()
        count += s.size
    return total / count


def test_psnr_known_answers():
    """test_metrics.cpp:80-85"""
    a = np.full((8, 8, 3), 0.3)
    assert math.isinf(O.psnr(a, a))
    assert O.psnr(np.zeros((8, 8, 3)), np.full((8, 8, 3), 0.1)) == pytest.approx(20.0, rel=1e-12)
    with pytest.raises(ValueError):
        O.psnr(np.zeros((4, 4, 3)), np.zeros((4, 5, 3)))


def test_ssim_properties():
    """test_metrics.cpp:101-150"""
    g = np.random.default_rng(52)
    a = g.uniform(size=(16, 16, 3))
    assert O.ssim(a, a) == pytest.approx(1.0, rel=1e-12)
    yy, xx = np.mgrid[0:16, 0:16]
    ck = ((xx + yy) % 2).astype(float)[:, :, None].repeat(3, 2)
    assert O.ssim(ck, 1.0 - ck) < 0.0
    for _ in range(5):
        a, b = g.uniform(size=(15, 20, 3)), g.uniform(size=(15, 20, 3))
        assert O.ssim(a, b) == pytest.approx(ssim_ref(a, b), rel=1e-6)
        assert abs(O.ssim(a, b) - O.ssim(b, a)) < 1e-12
    with pytest.raises(ValueError):
        O.ssim(np.zeros((12, 10, 3)), np.zeros((12, 10, 3)))


def test_ssim_and_loss_gradients_fd():
    """test_metrics.cpp:152-187"""
    g = np.random.default_rng(55)
    a, b = g.uniform(size=(13, 14, 3)), g.uniform(size=(13, 14, 3))
    _, grad = O.ssim_with_grad(a, b)
    h = 1e-6
    for _ in range(30):
        i = tuple(g.integers(0, s) for s in a.shape)
        ap, am = a.copy(), a.copy()
        ap[i] += h
        am[i] -= h
        fd = (O.ssim(ap, b) - O.ssim(am, b)) / (2 * h)
        assert grad[i] == pytest.approx(fd, rel=1e-4, abs=1e-10)
    gt, half = np.zeros((16, 16, 3)), np.full((16, 16, 3), 0.5)
    assert O.photometric_loss(gt, gt, 0.2) == 0.0
    assert O.photometric_loss(half, gt, 0.0) == pytest.approx(0.5, rel=1e-12)
    a, b = g.uniform(size=(16, 16, 3)), g.uniform(size=(16, 16, 3))
    loss, grad = O.photometric_loss_with_grad(a, b, 0.2)
    assert loss == pytest.approx(O.photometric_loss(a, b, 0.2), rel=1e-12)
    for _ in range(25):
        i = tuple(g.integers(0, s) for s in a.shape)
        ap, am = a.copy(), a.copy()
        ap[i] += h
        am[i] -= h
        fd = (O.photometric_loss(ap, b, 0.2) - O.photometric_loss(am, b, 0.2)) / (2 * h)
        assert grad[i] == pytest.approx(fd, rel=1e-4)


# ------------------------------------------------------------------ Adam
def one_of_each():
    """test_train.cpp:35-55"""
    s = HybridScene(sh_degree=1, extent=2.0)
    s.mean3 = np.array([[0.3, -0.2, 0.1]])
    s.quat3 = np.array([[1.0, 0, 0, 0]])
    s.log_s3 = np.array([[-1.0, -1.2, -0.9]])
    s.op3 = np.array([0.4])
    s.sh3 = np.zeros((1, 4, 3))
    s.sh3[0, 0] = [0.2, 0.3, 0.4]
    s.mean_x = np.array([[-0.1, 0.2, 0.4]])
    s.mean_t = np.array([0.5])
    s.ql = np.array([[1.0, 0, 0, 0]])
    s.qr = np.array([[1.0, 0, 0, 0]])
    s.log_s4 = np.array([[-1.1, -1.0, -0.8, math.log(0.07)]])
    s.op4 = np.array([-0.3])
    s.sh4 = np.zeros((1, 4, 3))
    s.sh4[0, 0] = [0.5, 0.1, 0.6]
    return s


class RefAdam:  # test_train.cpp:23-32
    def __init__(self):
        self.m = self.v = 0.0

    def step(self, value, grad, lr, t):
        self.m = 0.9 * self.m + 0.1 * grad
        self.v = 0.999 * self.v + (1 - 0.999) * grad * grad
        bc1, bc2 = 1 - 0.9 ** t, 1 - 0.999 ** t
        return value - lr * (self.m / bc1) / (math.sqrt(self.v / bc2) + 1e-15)


def test_adam_matches_scalar_reference():
    """test_train.cpp:71-111"""
    s = one_of_each()
    st = O.AdamState(s)
    lrs = O.LearningRates()
    g = np.random.default_rng(91)
    refs = [RefAdam() for _ in range(5)]
    vals = [s.mean3[0, 0], s.log_s3[0, 2], s.op4[0], s.sh3[0, 1, 2], s.mean_t[0]]
    for it in range(1, 6):
        gr = O.zero_grads(s)
        d = g.standard_normal(5)
        gr["mean3"][0, 0], gr["log_s3"][0, 2], gr["op4"][0], gr["sh3"][0, 1, 2], gr["mean_t"][0] = d
        O.optimizer_step(s, gr, st, lrs, 0.7)
        lr = [lrs.mean * s.extent * 0.7, lrs.scales, lrs.opacity, lrs.sh, lrs.mean_t * 0.7]
        vals = [refs[k].step(vals[k], d[k], lr[k], it) for k in range(5)]
        got = [s.mean3[0, 0], s.log_s3[0, 2], s.op4[0], s.sh3[0, 1, 2], s.mean_t[0]]
        for a, b in zip(got, vals):
            assert a == pytest.approx(b, rel=1e-12)
    assert st.step == 5


def test_quaternions_unit_and_canonical():
    """test_train.cpp:113-136"""
    rng = O.Rng(92)
    s = one_of_each()
    s.quat3[0], s.ql[0], s.qr[0] = rng.random_quat(), rng.random_quat(), rng.random_quat()
    st = O.AdamState(s)
    g = np.random.default_rng(92)
    for _ in range(20):
        gr = O.zero_grads(s)
        gr["quat3"][0], gr["ql"][0], gr["qr"][0] = 5 * g.standard_normal((3, 4))
        O.optimizer_step(s, gr, st)
        for q in (s.quat3[0], s.ql[0], s.qr[0]):
            assert np.linalg.norm(q) == pytest.approx(1.0, rel=1e-12)
            assert q[0] >= 0.0


def test_nonfinite_skips_row_only():
    """test_train.cpp:138-151"""
    s = one_of_each()
    st = O.AdamState(s)
    gr = O.zero_grads(s)
    gr["mean3"][0, 1] = np.nan
    gr["op3"][0] = 1.0
    m0, o0 = s.mean3.copy(), s.op3[0]
    O.optimizer_step(s, gr, st)
    assert (s.mean3 == m0).all() and s.op3[0] != o0
    assert st.skipped_nonfinite == 1


# ------------------------------------------------------------------ conversion
def test_is_static_strict():
    """test_scene.cpp:12-21"""
    tau = 0.7
    assert not O.is_static(math.log(tau), tau)
    assert O.is_static(math.log(tau) + 0.01, tau)
    assert not O.is_static(math.log(tau) - 0.01, tau)
    with pytest.raises(ValueError):
        O.is_static(0.0, 0.0)


def test_conversion_identity_pair_folds_mean_weight():
    """test_scene.cpp:23-50 (trapezoid integration known answer, 1e-9)"""
    ls4 = np.array([0.1, -0.2, 0.3, 0.9])
    m3, q3, ls3, op3 = O.convert_4d_to_3d([1.0, -2.0, 0.5], 0.3, [1, 0, 0, 0], [1, 0, 0, 0], ls4, 1.7)
    assert (m3 == [1.0, -2.0, 0.5]).all()
    assert np.abs(q3 - [1, 0, 0, 0]).max() < 1e-12
    assert (ls3 == ls4[:3]).all()
    sigma = math.exp(0.9)
    n = 200000
    t = np.arange(n + 1) / n
    w = np.exp(-0.5 * (t - 0.3) ** 2 / sigma ** 2)
    acc = w.sum() - 0.5 * (w[0] + w[-1])
    expected = 1 / (1 + math.exp(-1.7)) * acc / n
    assert 1 / (1 + math.exp(-op3)) == pytest.approx(expected, rel=1e-9)
    assert op3 < 1.7


def test_conversion_wide_limit_bit_exact():
    """test_scene.cpp:52-57"""
    _, _, _, op3 = O.convert_4d_to_3d([0, 0, 0], 0.5, [1, 0, 0, 0], [1, 0, 0, 0],
                                      [0, 0, 0, math.log(1e8)], -0.37)
    assert op3 == -0.37


def pair_from_rot4(rot):
    """gauss_math.cpp:123-152 (test-side helper: SO(4) -> isoclinic pair)."""
    def L(q):
        a, b, c, d = q
        return np.array([[a, -b, -c, -d], [b, a, -d, c], [c, d, a, -b], [d, -c, b, a]])

    def R(q):
        p, qq, r, s = q
        return np.array([[p, -qq, -r, -s], [qq, p, s, -r], [r, -s, p, qq], [s, r, -qq, p]])
    outer = np.zeros((4, 4))
    E = np.eye(4)
    for a in range(4):
        for b in range(4):
            outer[a, b] = 0.25 * (rot * (L(E[a]) @ R(E[b]))).sum()
    u, _, vt = np.linalg.svd(outer)
    ql, qr = u[:, 0], vt[0]
    if ql[0] < 0:
        ql = -ql
    if qr[0] < 0:
        qr = -qr
    if np.abs(L(ql) @ R(qr) - rot).max() > 1e-6:
        qr = -qr
    return ql, qr


def test_block_diagonal_converts_exactly():
    """test_scene.cpp:59-73"""
    rng = O.Rng(31)
    for _ in range(50):
        r3 = O.quat_to_rot3(rng.random_quat())
        embed = np.eye(4)
        embed[:3, :3] = r3
        ql, qr = pair_from_rot4(embed)
        assert np.abs(O.rot4_from_pair(ql, qr) - embed).max() < 1e-9
        _, q3, _, _ = O.convert_4d_to_3d([0, 0, 0], 0.5, ql, qr, [0, 0, 0, 0], 0.0)
        assert np.abs(O.quat_to_rot3(q3) - r3).max() < 1e-8


def test_low_leakage_conversion_renders_like_slice():
    """test_scene.cpp:75-115"""
    rng = O.Rng(32)
    cam = O.look_at([0, 0, -4], [0, 0, 0], [0, -1, 0], 60.0, 32, 32)
    tested = 0
    for _ in range(40):
        if tested >= 5:
            break
        embed = np.eye(4)
        embed[:3, :3] = O.quat_to_rot3(rng.random_quat())
        th = 0.004
        mix = np.eye(4)
        mix[0, 0], mix[0, 3], mix[3, 0], mix[3, 3] = math.cos(th), -math.sin(th), math.sin(th), math.cos(th)
        ql, qr = pair_from_rot4(embed @ mix)
        ls4 = np.array([math.log(0.4), math.log(0.3), math.log(0.35), math.log(2.0)])
        _, leak = O.extract_spatial_rot(O.rot4_from_pair(ql, qr))
        if leak >= 0.05:
            continue
        tested += 1
        sh = ((np.array([0.8, 0.4, 0.2]) - 0.5) / C0).reshape(1, 1, 3)
        s4 = HybridScene(sh_degree=0, mean_x=[[0.1, -0.1, 0.0]], mean_t=[0.5], ql=[ql], qr=[qr],
                         log_s4=[ls4], op4=[logit(0.8)], sh4=sh)
        m3, q3, ls3, op3 = O.convert_4d_to_3d([0.1, -0.1, 0.0], 0.5, ql, qr, ls4, logit(0.8))
        s3 = HybridScene(sh_degree=0, mean3=[m3], quat3=[q3], log_s3=[ls3], op3=[op3], sh3=sh)
        a = O.rasterize(s4, cam, 0.5)["rgb"]
        b = O.rasterize(s3, cam, 0.5)["rgb"]
        assert np.abs(a - b).max() < 0.01
    assert tested >= 5


def test_sweep_moves_exactly_above_threshold_in_order():
    """test_scene.cpp:117-140"""
    rng = O.Rng(33)
    s = rng.random_scene(3, 20)
    s.tau = 0.3
    scales = np.exp(s.log_s4[:, 3])
    moved, rep = O.sweep_convert(s)
    expected = np.nonzero(scales > s.tau)[0]
    assert (moved == expected).all()
    assert rep["count"] == len(expected)
    assert s.n3 == 3 + len(expected) and s.n4 == 20 - len(expected)
    assert not (np.exp(s.log_s4[:, 3]) > s.tau).any()
    assert rep["max_leakage"] >= rep["mean_leakage"]
    again, rep2 = O.sweep_convert(s)
    assert rep2["count"] == 0 and len(again) == 0


def test_sweep_remaps_optimizer_rows():
    """train.cpp:305-362: converted rows inherit mean_x, scales[:3], quat_left,
    opacity and SH moments; survivors keep order; all stats reset."""
    rng = O.Rng(34)
    s = rng.random_scene(2, 12)
    s.tau = 0.3
    st = O.AdamState(s)
    g = np.random.default_rng(0)
    for b in (st.m, st.v):
        for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
            getattr(b, f)[...] = g.standard_normal(getattr(b, f).shape)
    st.grad_norm4[:] = 1.0
    st.count4[:] = 3
    m_before = st.m.copy()
    mask = np.exp(s.log_s4[:, 3]) > s.tau
    moved, _ = O.sweep_convert(s, st)
    assert (moved == np.nonzero(mask)[0]).all()
    k = len(moved)
    assert (st.m.mean3[2:] == m_before.mean_x[moved]).all()
    assert (st.m.log_s3[2:] == m_before.log_s4[moved, :3]).all()
    assert (st.m.quat3[2:] == m_before.ql[moved]).all()
    assert (st.m.op3[2:] == m_before.op4[moved]).all()
    assert (st.m.sh3[2:] == m_before.sh4[moved]).all()
    assert (st.m.mean3[:2] == m_before.mean3).all()
    keep = np.nonzero(~mask)[0]
    assert (st.m.qr == m_before.qr[keep]).all()
    assert st.grad_norm4.shape == (12 - k,) and (st.grad_norm4 == 0).all() and (st.count3 == 0).all()
