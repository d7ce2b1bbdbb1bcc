"""Pins the oracle's math kernels against the reference's own tests.

Restates include/hgs tests test_gauss_math.cpp and test_sh.cpp (file:line in
each test docstring).  The reference cannot be built here, so
these property / closed-form tests are what pins the oracle.  Random draws use
numpy for pure property checks (the exact draw sequence of a property test is
immaterial); seeded scene fixtures use the oracle's libstdc++ mt19937_64.
"""
import math

import numpy as np
import pytest

import oracle as O


def quat_mul(a, b):  # tests/oracles.hpp:19-24
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


def is_rotation(m, tol):
    return np.abs(m.T @ m - np.eye(len(m))).max() <= tol and abs(np.linalg.det(m) - 1) <= tol


def test_quat_rot_roundtrip():
    """test_gauss_math.cpp:25-34"""
    rng = O.Rng(11)
    for _ in range(500):
        q = rng.random_quat()
        r = O.quat_to_rot3(q)
        assert is_rotation(r, 1e-12)
        assert np.abs(O.rot3_to_quat(r) - q).max() < 1e-9


def test_rot3_to_quat_trace_minus_one_branch():
    """test_gauss_math.cpp:36-48"""
    g = np.random.default_rng(12)
    for _ in range(200):
        ax = g.standard_normal(3)
        ax /= np.linalg.norm(ax)
        q = np.array([0.0, *ax])
        n = np.sqrt((q * q).sum())
        q /= n
        for k in range(1, 4):  # canonical sign with w == 0
            if q[k] != 0:
                if q[k] < 0:
                    q = -q
                break
        r = O.quat_to_rot3(q)
        assert np.abs(O.rot3_to_quat(r) - q).max() < 1e-9
    with pytest.raises(ValueError):
        O.rot3_to_quat(2.0 * np.eye(3))


def test_isoclinic_matches_quaternion_product():
    """test_gauss_math.cpp:50-70"""
    rng = O.Rng(13)
    g = np.random.default_rng(13)
    for _ in range(300):
        ql, qr = rng.random_quat(), rng.random_quat()
        rot = O.rot4_from_pair(ql, qr)
        assert is_rotation(rot, 1e-12)
        x = g.standard_normal(4)
        via = quat_mul(ql, quat_mul(x, qr))
        assert np.abs(rot @ x - via).max() < 1e-12 * (1 + np.linalg.norm(x))
    assert np.abs(O.rot4_from_pair([1, 0, 0, 0], [1, 0, 0, 0]) - np.eye(4)).max() == 0.0


def test_covariance_symmetric_psd_with_exp2s_spectrum():
    """test_gauss_math.cpp:85-111"""
    rng = O.Rng(15)
    g = np.random.default_rng(15)
    for _ in range(200):
        ql, qr = rng.random_quat(), rng.random_quat()
        ls = g.uniform(-2.0, 1.0, 4)
        cov = O.build_cov4(O.rot4_from_pair(ql, qr), ls)
        assert np.abs(cov - cov.T).max() == 0.0  # exactly symmetric by construction
        ev = np.linalg.eigvalsh(cov)
        exp = np.sort(np.exp(2 * ls))
        assert np.abs(ev - exp).max() < 1e-9 * exp.max()
        c3 = O.build_cov3(O.quat_to_rot3(ql), ls[:3])
        assert np.abs(c3 - c3.T).max() < 1e-12


def test_clamp_psd():
    """test_gauss_math.cpp:113-129"""
    asym = np.array([[1.0, 0.2, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    s = O.clamp_psd(asym)
    assert np.abs(s - s.T).max() == 0.0
    nearly = np.eye(3)
    nearly[2, 2] = -5e-9
    c = O.clamp_psd(nearly)
    assert np.linalg.eigvalsh(c).min() >= 1e-12 * (1 - 1e-9)
    bad = np.eye(3)
    bad[2, 2] = -1.0
    with pytest.raises(ValueError):
        O.clamp_psd(bad)


def test_condition_matches_precision_oracle():
    """test_gauss_math.cpp:131-148 (condition_via_precision, oracles.hpp:48-59)"""
    g = np.random.default_rng(16)
    for _ in range(1000):
        a = g.standard_normal((4, 4))
        cov = a @ a.T + 1e-3 * np.eye(4)
        mean = np.array([g.standard_normal(), g.standard_normal(), g.standard_normal(), g.uniform()])
        t = g.uniform()
        m3, c3, w = O.condition_at_time(mean, cov, t)
        prec = np.linalg.inv(cov)
        ref_cov = np.linalg.inv(prec[:3, :3])
        ref_mean = mean[:3] - ref_cov @ prec[:3, 3] * (t - mean[3])
        ref_w = math.exp(-0.5 * (t - mean[3]) ** 2 / cov[3, 3])
        scale = np.abs(cov).max()
        assert np.abs(m3 - ref_mean).max() < 1e-10 * (1 + scale)
        assert np.abs(c3 - ref_cov).max() < 1e-10 * (1 + scale)
        assert w == pytest.approx(ref_w, rel=1e-12)
        assert 0.0 < w <= 1.0


def test_condition_at_mean_time_and_block_diagonal():
    """test_gauss_math.cpp:150-169 (known answer exp(-0.5*0.09/0.09))"""
    g = np.random.default_rng(17)
    a = g.standard_normal((4, 4))
    cov = a @ a.T + 1e-3 * np.eye(4)
    mean = np.array([0.3, -0.2, 0.9, 0.4])
    m3, _, w = O.condition_at_time(mean, cov, 0.4)
    assert np.abs(m3 - mean[:3]).max() == 0.0 and w == 1.0
    cov = np.zeros((4, 4))
    cov[:3, :3] = [[0.4, 0.1, 0.0], [0.1, 0.3, 0.05], [0.0, 0.05, 0.2]]
    cov[3, 3] = 0.09
    m3, c3, w = O.condition_at_time(np.array([1.0, 2.0, 3.0, 0.5]), cov, 0.8)
    assert np.abs(m3 - [1, 2, 3]).max() < 1e-15
    assert np.abs(c3 - cov[:3, :3]).max() < 1e-12
    assert w == pytest.approx(math.exp(-0.5 * 0.3 * 0.3 / 0.09), rel=1e-12)


def test_degenerate_temporal_rejected():
    """test_gauss_math.cpp:171-175"""
    cov = np.eye(4)
    cov[3, 3] = 1e-13
    with pytest.raises(O.DegenerateTemporalError):
        O.condition_at_time(np.zeros(4), cov, 0.5)


def test_extract_spatial_rot_polar_optimal():
    """test_gauss_math.cpp:177-198"""
    rng = O.Rng(18)
    for _ in range(200):
        rot = O.rot4_from_pair(rng.random_quat(), rng.random_quat())
        r3, leak = O.extract_spatial_rot(rot)
        assert is_rotation(r3, 1e-9)
        block = rot[:3, :3]
        best = np.trace(r3.T @ block)
        for _ in range(20):
            other = O.quat_to_rot3(rng.random_quat())
            assert np.trace(other.T @ block) <= best + 1e-9
        exp = math.sqrt((rot[:3, 3] ** 2).sum() + (rot[3, :3] ** 2).sum())
        assert leak == pytest.approx(exp, rel=1e-12)


def test_block_diagonal_rotation_extracts_exactly():
    """test_gauss_math.cpp:200-208"""
    rng = O.Rng(19)
    r3 = O.quat_to_rot3(rng.random_quat())
    rot = np.eye(4)
    rot[:3, :3] = r3
    got, leak = O.extract_spatial_rot(rot)
    assert np.abs(got - r3).max() < 1e-12
    assert leak == 0.0


# ------------------------------------------------------------------ SH
C0 = 0.28209479177387814
C1 = 0.4886025119029199


def test_sh_closed_form():
    """test_sh.cpp:47-59 (real SH closed forms) and 99-108 (band 1 known answer)"""
    g = np.random.default_rng(3)
    for _ in range(100):
        d = g.standard_normal(3)
        d /= np.linalg.norm(d)
        x, y, z = d
        b = O.sh_basis(d, 3)
        exp = [C0, -C1 * y, C1 * z, -C1 * x,
               1.0925484305920792 * x * y, -1.0925484305920792 * y * z,
               0.31539156525252005 * (2 * z * z - x * x - y * y), -1.0925484305920792 * x * z,
               0.5462742152960396 * (x * x - y * y),
               -0.5900435899266435 * y * (3 * x * x - y * y), 2.890611442640554 * x * y * z,
               -0.4570457994644658 * y * (4 * z * z - x * x - y * y),
               0.3731763325901154 * z * (2 * z * z - 3 * x * x - 3 * y * y),
               -0.4570457994644658 * x * (4 * z * z - x * x - y * y),
               1.445305721320277 * z * (x * x - y * y), -0.5900435899266435 * x * (x * x - 3 * y * y)]
        assert np.abs(b - exp).max() < 1e-12
    b = O.sh_basis([1.0, 0.0, 0.0], 1)
    assert b[3] == pytest.approx(-0.4886025119029199, abs=1e-15)


def test_sh_basis_grad_fd():
    """test_sh.cpp:61-81"""
    g = np.random.default_rng(4)
    h = 1e-6
    for _ in range(40):
        d = g.standard_normal(3)
        gr = O.sh_basis_grad(d, 3)
        for c in range(3):
            dp, dm = d.copy(), d.copy()
            dp[c] += h
            dm[c] -= h
            fd = (O.sh_basis(dp, 3) - O.sh_basis(dm, 3)) / (2 * h)
            assert np.abs(fd - gr[:, c]).max() < 1e-6


def test_eval_sh_dc_roundtrip_and_clamp():
    """test_sh.cpp:83-92"""
    rgb = np.array([0.2, 0.5, 0.9])
    coeffs = np.zeros((4, 3))
    coeffs[0] = (rgb - 0.5) / C0
    out = O.eval_sh(coeffs, 1, [0.0, 0.0, 1.0])
    assert np.abs(out - rgb).max() < 1e-12
    coeffs[0] = (np.array([2.0, -1.0, 0.5]) - 0.5) / C0
    out = O.eval_sh(coeffs, 1, [0.0, 0.0, 1.0])
    assert out[0] == 1.0 and out[1] == 0.0
    with pytest.raises(ValueError):
        O.eval_sh(coeffs, 1, [0.0, 0.0, 2.0])
