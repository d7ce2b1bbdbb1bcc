"""The C-ABI multi-GPU exchange (hgs_comm_*, hgs_allreduce_grads,
hgs_param_checksum, hgs_broadcast_params) on one B200: a one-rank NCCL
communicator exercises the whole plumbing (the grouped in-place
ncclAllReduce of every gradient row on the context stream) with the identity
reduction; two processes sharing the GPU exchange through gloo in
tests/test_gpu_dist_product.py (NCCL refuses two ranks on one device), and the
multi-rank host logic is covered by tests/test_dist_cpu.py."""
import numpy as np
import pytest

from paper_2505_13215_b200 import api as A
from paper_2505_13215_b200.scene import ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu


def _trainer(ctx, exchange=None):
    from paper_2505_13215_b200.train import DeviceTrainer

    target = synthetic_scene(3000, 2000, sh_degree=2, seed=31)
    scene = synthetic_scene(3000, 2000, sh_degree=2, seed=32).as_float32_exact()
    cams = [ring_camera(i, 96, 72) for i in range(4)]
    return DeviceTrainer(ctx, scene, cams, [0.1, 0.4, 0.6, 0.9], target=target, iterations=50)


def test_one_rank_allreduce_is_identity():
    with A.Context(0) as ctx:
        tr = _trainer(ctx)
        uid = A.Context.comm_unique_id()
        assert len(uid) == 128
        ctx.comm_init(1, 0, uid)
        assert ctx._lib.hgs_comm_size(ctx.handle) == 1
        tr.step([0, 1], apply_adam=False)
        before = ctx.grads()
        ctx.allreduce_grads()
        after = ctx.grads()
        for k in before:
            assert np.array_equal(np.asarray(before[k]), np.asarray(after[k])), k
        assert np.array_equal(ctx.allreduce_f64([1.5, -2.0, np.inf]), [1.5, -2.0, np.inf])
        s0 = ctx.param_checksum()
        ctx.broadcast_params(0)
        assert ctx.param_checksum() == s0
        ctx.adam_step(tr.lrs, tr.decay())
        assert ctx.param_checksum() != s0
        ctx.comm_destroy()
        with pytest.raises(A.StateError):
            ctx.allreduce_grads()


def test_param_checksum_detects_one_flipped_value():
    scene = synthetic_scene(5000, 3000, sh_degree=3, seed=3).as_float32_exact()
    with A.Context(0) as a, A.Context(0) as b:
        a.upload(scene)
        b.upload(scene)
        assert a.param_checksum() == b.param_checksum()
        s2 = scene.copy()
        s2.sh3[1234, 7, 2] = np.nextafter(np.float32(s2.sh3[1234, 7, 2]), np.float32(1)).astype(np.float64)
        b.upload(s2)
        assert a.param_checksum() != b.param_checksum()
        s3 = scene.copy()  # the same multiset of values in another order is another scene
        s3.op4[[0, 1]] = s3.op4[[1, 0]]
        b.upload(s3)
        assert (s3.op4[0] == s3.op4[1]) or a.param_checksum() != b.param_checksum()


def test_view_parallel_trainer_capi_exchange_single_rank(tmp_path):
    """ViewParallelTrainer(exchange='capi') in a one-rank process group: the
    same iteration as the plain trainer (FP32 tolerance: atomics)."""
    import os

    import torch.distributed as dist

    from paper_2505_13215_b200.train import ViewParallelTrainer

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29617")
    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"file://{tmp_path}/pg")
    try:
        target = synthetic_scene(3000, 2000, sh_degree=2, seed=31)
        scene = synthetic_scene(3000, 2000, sh_degree=2, seed=32).as_float32_exact()
        cams = [ring_camera(i, 96, 72) for i in range(4)]
        times = [0.1, 0.4, 0.6, 0.9]
        with A.Context(0) as c1, A.Context(0) as c2:
            from paper_2505_13215_b200.train import DeviceTrainer

            ref = DeviceTrainer(c1, scene, cams, times, target=target, iterations=50)
            vp = ViewParallelTrainer(c2, scene, cams, times, target=target, iterations=50, exchange="capi",
                                     verify_every=1)
            for it in range(3):
                l1 = ref.step([it % 4, (it + 1) % 4])
                l2 = vp.step([it % 4, (it + 1) % 4])
                assert l2 == pytest.approx(l1, rel=1e-5)
            assert vp.repairs == 0
            s1, s2 = c1.download(), c2.download()
            for f in ("mean_x", "log_s4", "sh4", "mean3", "op3"):
                np.testing.assert_allclose(getattr(s2, f), getattr(s1, f), rtol=1e-4, atol=1e-6)
    finally:
        dist.destroy_process_group()


def test_pipelined_exchange_single_rank(tmp_path):
    """hgs_train_exchange_async (ViewParallelTrainer.step_async): pipelined
    view-parallel iterations with the all-reduced loss gate -- the same
    iterations as the plain trainer; a non-finite batch raises NumericAbort
    at its collect and leaves the parameters untouched."""
    import torch
    import torch.distributed as dist

    from paper_2505_13215_b200.train import DeviceTrainer, ViewParallelTrainer

    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"file://{tmp_path}/pg2")
    try:
        target = synthetic_scene(3000, 2000, sh_degree=2, seed=41)
        scene = synthetic_scene(3000, 2000, sh_degree=2, seed=42).as_float32_exact()
        cams = [ring_camera(i, 96, 72) for i in range(4)]
        times = [0.1, 0.4, 0.6, 0.9]
        with A.Context(0) as c1, A.Context(0) as c2:
            ref = DeviceTrainer(c1, scene, cams, times, target=target, iterations=50)
            vp = ViewParallelTrainer(c2, scene, cams, times, target=target, iterations=50, exchange="capi")
            batches = [[it % 4, (it + 1) % 4] for it in range(6)]
            want = [ref.step(b) for b in batches]
            got = []
            for b in batches:
                vp.step_async(b)
                if c2._lib.hgs_train_pending(c2.handle) > 2:
                    got.append(vp.collect())
            while c2._lib.hgs_train_pending(c2.handle):
                got.append(vp.collect())
            assert got == pytest.approx(want, rel=1e-5)
            s1, s2 = c1.download(), c2.download()
            for f in ("mean_x", "ql", "log_s4", "sh4", "mean3", "op3"):
                np.testing.assert_allclose(getattr(s2, f), getattr(s1, f), rtol=1e-4, atol=1e-6)
            # a non-finite batch: NumericAbort at its collect, parameters untouched
            before = c2.download()
            vp.gt[1] = torch.full_like(vp.gt[1], float("nan"))
            vp.step_async([0, 1])
            with pytest.raises(A.NumericAbort):
                vp.collect()
            after = c2.download()
            for f in ("mean_x", "sh4", "op3"):
                assert np.array_equal(getattr(after, f), getattr(before, f)), f
            vp.step_async([2, 3])  # the gate re-arms
            assert np.isfinite(vp.collect())
    finally:
        dist.destroy_process_group()


def test_exchange_binds_the_process_nccl():
    """In a process where torch.distributed already mapped its NCCL, the
    library's exchange binds that same copy (one NCCL per process)."""
    import ctypes as C

    import torch

    from paper_2505_13215_b200 import _capi

    torch.cuda.init()
    import torch.distributed  # noqa: F401  (maps torch's libnccl)

    ver = C.c_int()
    buf = C.create_string_buffer(512)
    assert _capi.lib().hgs_comm_nccl_info(C.byref(ver), buf, 512) == 0
    tv = torch.cuda.nccl.version()
    tcode = tv[0] * 10000 + tv[1] * 100 + tv[2] if isinstance(tv, tuple) else int(tv)
    assert ver.value == tcode, (ver.value, tcode, buf.value)


def test_sharded_exchange_one_rank_matches_the_allreduce_exchange(tmp_path):
    """hgs_comm_set_sharded: reduce-scatter -> Adam on the rank's shard ->
    all-gather.  With a one-rank communicator the shard is the whole pool:
    three pipelined exchange steps give the parameters and moments of the
    all-reduce exchange (FP tolerance: K6's atomics order), the moments are
    flagged sharded until hgs_gather_state, and the state-dependent calls
    refuse to run on sharded moments."""
    import ctypes as C

    from paper_2505_13215_b200.train import DeviceTrainer

    with A.Context(0) as a, A.Context(0) as b:
        ta, tb = _trainer(a), _trainer(b)
        for ctx in (a, b):
            ctx.comm_init(1, 0, A.Context.comm_unique_id())
        b.set_sharded(True)
        for i in range(3):
            for ctx, tr in ((a, ta), (b, tb)):
                DeviceTrainer.step_async(tr, [i % 4], batch_total=1, apply_adam=False)
                ctx._check(ctx._lib.hgs_train_exchange_async(ctx.handle, C.byref(tr._opts(tr.decay()))))
                tr.collect()
        sa, sb = a.download(), b.download()
        for f in ("mean_x", "ql", "log_s4", "op4", "sh4", "mean3", "quat3", "op3", "sh3"):
            x, y = np.asarray(getattr(sa, f)), np.asarray(getattr(sb, f))
            assert np.allclose(x, y, rtol=1e-5, atol=1e-7), f
        with pytest.raises(A.StateError):
            b.save_checkpoint(str(tmp_path / "s.hgsc"))
        with pytest.raises(A.StateError):
            b.sweep_convert()
        b.gather_state()
        ma, va = a.adam_state()[:2]
        mb, vb = b.adam_state()[:2]
        for f in ("mean_x", "sh4", "mean3", "sh3"):
            assert np.allclose(np.asarray(getattr(ma, f)), np.asarray(getattr(mb, f)), rtol=1e-4, atol=1e-9), f
            assert np.allclose(np.asarray(getattr(va, f)), np.asarray(getattr(vb, f)), rtol=1e-4, atol=1e-12), f
        b.save_checkpoint(str(tmp_path / "s.hgsc"))
        assert np.array_equal(a.densify_stats()[0], b.densify_stats()[0]) or np.allclose(
            a.densify_stats()[0], b.densify_stats()[0], rtol=1e-5)
