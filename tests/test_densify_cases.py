"""The reference's densify_and_prune unit tests (test_train.cpp:153-233)
restated on the oracle (CPU) and on the device (GPU: the case is loaded as a
checkpoint -- scene, Adam moments and statistics -- then
hgs_densify_and_prune runs with the same libstdc++ seed)."""
import math

import numpy as np
import pytest

import oracle as O
from oracle import checkpoint as CK
from paper_2505_13215_b200.scene import HybridScene

FIELDS = HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS
CFG = dict(grad_threshold=0.02, opacity_prune_eps=0.005, clone_size_frac=0.01, split_factor=1.6,
           max_gaussians=20000)  # TrainConfig defaults (train.hpp:23-49)


def logit(p):
    return math.log(p / (1.0 - p))


def one_of_each(n3=1):
    """test_train.cpp:25-45"""
    s = HybridScene(sh_degree=1, extent=2.0,
                    mean3=[[0.3, -0.2, 0.1]] * n3, quat3=[[1.0, 0, 0, 0]] * n3, log_s3=[[-1.0, -1.2, -0.9]] * n3,
                    op3=[0.4] * n3,
                    mean_x=[[-0.1, 0.2, 0.4]], mean_t=[0.5], ql=[[1.0, 0, 0, 0]], qr=[[1.0, 0, 0, 0]],
                    log_s4=[[-1.1, -1.0, -0.8, math.log(0.07)]], op4=[-0.3])
    s.sh3[:, 0, :] = [0.2, 0.3, 0.4]
    s.sh4[:, 0, :] = [0.5, 0.1, 0.6]
    return s


def state_for(scene):
    st = O.AdamState(scene)
    return st


def case_prune():
    s = one_of_each(2)
    s.op3[0] = logit(0.001)  # below the prune threshold
    s.op3[1] = logit(0.5)
    st = state_for(s)
    st.m.mean3[1, 0] = 7.5  # the survivor's row moves to row 0
    st.m.mean3[0, 0] = -1.0
    return s, st, dict(CFG), 93


def case_clone():
    s = one_of_each()
    s.extent = 10.0
    s.log_s3[0] = [math.log(0.01)] * 3  # below the size gate
    st = state_for(s)
    st.m.mean3[0, 0] = 3.25
    st.grad_norm3[0], st.count3[0] = 1.0, 2  # avg 0.5 > threshold
    return s, st, dict(CFG, grad_threshold=0.02, clone_size_frac=0.01), 94


def case_split():
    s = one_of_each()
    s.extent = 1.0
    s.log_s4[0, :3] = math.log(0.5)  # above the gate
    st = state_for(s)
    st.grad_norm4[0], st.count4[0] = 1.0, 1
    return s, st, dict(CFG), 95


def case_cap():
    s = one_of_each()
    s.log_s3[0] = [math.log(0.001)] * 3
    st = state_for(s)
    st.grad_norm3[0], st.count3[0] = 1.0, 1
    return s, st, dict(CFG, max_gaussians=1), 96


CASES = {"prune": case_prune, "clone": case_clone, "split": case_split, "cap": case_cap}


def check_reference_expectations(name, s0, out, st, rep, cfg):
    if name == "prune":  # test_train.cpp:153-172
        assert rep["pruned3"] == 1 and out.n3 == 1
        assert st.m.mean3[0, 0] == 7.5
        assert st.grad_norm3.shape == (1,) and st.grad_norm3[0] == 0.0 and st.count3[0] == 0
    elif name == "clone":  # 174-195
        assert rep["cloned3"] == 1 and out.n3 == 2
        assert st.m.mean3[0, 0] == 3.25 and st.m.mean3[1, 0] == 0.0
        assert not np.array_equal(out.mean3[0], out.mean3[1])
        assert np.array_equal(out.log_s3[0], out.log_s3[1])
    elif name == "split":  # 197-218
        assert rep["split4"] == 1 and out.n4 == 2
        want = s0.log_s4[0] - math.log(cfg["split_factor"])
        for g in out.log_s4:
            assert np.abs(g - want).max() < 1e-6
        assert not st.m.log_s4.any()
    elif name == "cap":  # 220-233
        assert rep["cloned3"] == 0 and out.n3 == 1


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_densify_reference_cases(name):
    s, st, cfg, seed = CASES[name]()
    out, ost, rep = O.densify_and_prune(s, st, O.Rng(seed), **cfg)
    check_reference_expectations(name, s, out, ost, rep, cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_densify_reference_cases(name, tmp_path):
    from paper_2505_13215_b200 import api as A

    s, st, cfg, seed = CASES[name]()
    s = s.as_float32_exact()
    for f in FIELDS:  # the device holds FP32 moments
        getattr(st.m, f)[...] = getattr(st.m, f).astype(np.float32)
    p = str(tmp_path / "case.hgsc")
    CK.save_checkpoint(s, st, p)
    with A.Context(0) as ctx:
        assert ctx.load_checkpoint(p)
        rep = ctx.densify_and_prune(A.Rng(seed), **cfg)
        out = ctx.download()
        m, v, _ = ctx.adam_state()
        gn4, c4, gn3, c3 = ctx.densify_stats()
    dst = CK.State(out)
    dst.m, dst.v, dst.grad_norm3, dst.count3 = m, v, gn3, c3
    check_reference_expectations(name, s, out, dst, rep, cfg)
    ref, rst, rrep = O.densify_and_prune(s, st, O.Rng(seed), **cfg)
    for k in ("cloned3", "split3", "pruned3", "cloned4", "split4", "pruned4"):
        assert rep[k] == rrep[k], k
    for f in FIELDS:
        np.testing.assert_allclose(getattr(out, f), getattr(ref, f), rtol=1e-6, atol=1e-6, err_msg=f)
        np.testing.assert_allclose(getattr(m, f), getattr(rst.m, f), rtol=1e-6, atol=1e-7, err_msg=f)
