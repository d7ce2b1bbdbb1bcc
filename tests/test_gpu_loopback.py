"""The C-ABI exchange with TWO ranks on one B200, through the library's own
collective path (csrc/comm.cu), NCCL replaced by its in-process loopback
double (HGS_NCCL_LOOPBACK=1: ranks are threads of one process sharing the
device; every all-reduce / reduce-scatter / all-gather / broadcast is a host
barrier + a combine kernel in rank order).  NCCL itself refuses two ranks on
one device, so this is how the N > 1 product path -- hgs_train_exchange_async
with the grouped all-reduce, and the sharded reduce-scatter -> Adam on the
rank's shard -> all-gather -- runs here (2 ranks; the sharded exchange also
with 3, one of which renders no view).  Checked: the replicas are
bit-identical after three exchanged iterations in both modes, the sharded
exchange gives the all-reduce exchange's parameters and (after
hgs_gather_state) Adam moments, the replicas' summed loss equals one process
running the 2-view iteration, a non-finite loss on one rank aborts the same
iteration on every rank, and a broadcast repairs a diverged replica.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4", "mean3", "quat3", "log_s3", "op3", "sh3")


def _setup():
    from paper_2505_13215_b200.scene import ring_camera, synthetic_scene

    target = synthetic_scene(3001, 2003, sh_degree=3, seed=81)  # odd counts: ragged shards
    scene = synthetic_scene(3001, 2003, sh_degree=3, seed=82).as_float32_exact()
    cams = [ring_camera(8, 96, 72, index=i, n_ring=4) for i in range(4)]
    return scene, target, cams, [0.1, 0.4, 0.6, 0.9]


def _run_ranks(mode, world, out, errs, tmp):
    import ctypes as C
    import threading

    from paper_2505_13215_b200 import api as A
    from paper_2505_13215_b200.train import DeviceTrainer, shard_batch

    scene, target, cams, times = _setup()
    uid = A.Context.comm_unique_id()
    ctxs = [A.Context(0) for _ in range(world)]
    trs = [DeviceTrainer(c, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2), iterations=50) for c in ctxs]

    def rank_fn(r):
        try:
            ctx, tr = ctxs[r], trs[r]
            ctx.comm_init(world, r, uid)
            ctx.set_sharded(mode == "sharded")
            losses = []
            for i in range(3):
                batch = [i % 4, (i + 1) % 4]
                tr.iter += 1
                DeviceTrainer.step_async(tr, shard_batch(batch, r, world), batch_total=len(batch),
                                         apply_adam=False)
                ctx._check(ctx._lib.hgs_train_exchange_async(ctx.handle, C.byref(tr._opts(tr.decay()))))
                losses.append(tr.collect())
            refused = False  # sharded moments: the state-dependent calls refuse
            try:
                ctx.save_checkpoint(os.path.join(tmp, f"{mode}{world}_{r}.hgsc"))
            except A.StateError:
                refused = True
            ctx.gather_state()  # collective
            s = ctx.download()
            m, v, step = ctx.adam_state()
            out[(mode, world, r)] = dict(losses=losses, checksum=ctx.param_checksum(), step=step, refused=refused,
                                  p={f: np.asarray(getattr(s, f)).copy() for f in FIELDS},
                                  m={f: np.asarray(getattr(m, f)).copy() for f in FIELDS},
                                  v={f: np.asarray(getattr(v, f)).copy() for f in FIELDS},
                                  stats=[np.asarray(a).copy() for a in ctx.densify_stats()])
            if mode == "allreduce":
                # a diverged replica is repaired by a broadcast from rank 0
                if r == 1:
                    s2 = ctx.download()
                    s2.op3[:7] += 0.25
                    ctx.upload(s2)
                before = ctx.param_checksum()
                ctx.broadcast_params(0)
                out[(mode, world, r, "repair")] = (before, ctx.param_checksum())
        except BaseException as e:  # reported by the parent
            errs.append(f"{mode} rank {r}: {type(e).__name__}: {e}")

    ts = [threading.Thread(target=rank_fn, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for c in ctxs:
        c.close()


def _run_abort(mode, out, errs):
    """Rank 1's view of iteration 1 has a NaN ground-truth pixel: the
    exchanged loss gate makes every rank skip that update and raise
    NumericAbort for the same iteration (train.cpp:445-447); training then
    continues in lock step."""
    import ctypes as C
    import threading

    from paper_2505_13215_b200 import api as A
    from paper_2505_13215_b200._capi import NumericAbort
    from paper_2505_13215_b200.train import DeviceTrainer, shard_batch

    world = 2
    scene, target, cams, times = _setup()
    uid = A.Context.comm_unique_id()
    ctxs = [A.Context(0) for _ in range(world)]
    trs = [DeviceTrainer(c, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2), iterations=50) for c in ctxs]

    def rank_fn(r):
        try:
            ctx, tr = ctxs[r], trs[r]
            ctx.comm_init(world, r, uid)
            ctx.set_sharded(mode == "sharded")
            res = []
            for i in range(3):
                batch = [i % 4, (i + 1) % 4]
                mine = shard_batch(batch, r, world)
                poison = i == 1 and r == 1
                if poison:
                    tr.gt[mine[0]][3, 3, 0] = float("nan")
                tr.iter += 1
                DeviceTrainer.step_async(tr, mine, batch_total=len(batch), apply_adam=False)
                ctx._check(ctx._lib.hgs_train_exchange_async(ctx.handle, C.byref(tr._opts(tr.decay()))))
                try:
                    tr.collect()
                    res.append(("ok", ctx.param_checksum()))
                except NumericAbort:
                    tr._pending_n = []
                    res.append(("abort", ctx.param_checksum()))
                if poison:
                    tr.gt[mine[0]][3, 3, 0] = 0.5
            out[("abort", mode, r)] = res
        except BaseException as e:
            errs.append(f"abort {mode} rank {r}: {type(e).__name__}: {e}")

    ts = [threading.Thread(target=rank_fn, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for c in ctxs:
        c.close()


def _child(path):
    out, errs = {}, []
    for mode, world in (("allreduce", 2), ("sharded", 2), ("sharded", 3)):
        _run_ranks(mode, world, out, errs, os.path.dirname(path))
        if errs:
            break
    for mode in ("allreduce", "sharded"):
        if not errs:
            _run_abort(mode, out, errs)
    # one process, no exchange: the first 2-view iteration's loss
    from paper_2505_13215_b200.api import Context
    from paper_2505_13215_b200.train import DeviceTrainer

    ref_loss = None
    if not errs:
        scene, target, cams, times = _setup()
        with Context(0) as ctx:
            tr = DeviceTrainer(ctx, scene, cams, times, target=target, bg=(0.2, 0.2, 0.2), iterations=50)
            ref_loss = tr.step([0, 1], apply_adam=False)
    np.save(path, np.array([dict(out=out, errs=errs, ref_loss=ref_loss)], dtype=object), allow_pickle=True)


def test_two_rank_exchange_loopback(tmp_path):
    path = str(tmp_path / "loop.npy")
    old = os.environ.get("HGS_NCCL_LOOPBACK")
    os.environ["HGS_NCCL_LOOPBACK"] = "1"  # read by the child's library at its first collective
    try:
        p = mp.get_context("spawn").Process(target=_child, args=(path,))
        p.start()
        p.join(900)
    finally:
        if old is None:
            os.environ.pop("HGS_NCCL_LOOPBACK", None)
        else:
            os.environ["HGS_NCCL_LOOPBACK"] = old
    assert p.exitcode == 0, p.exitcode
    res = np.load(path, allow_pickle=True)[0]
    assert not res["errs"], res["errs"]
    out = res["out"]
    for mode, world in (("allreduce", 2), ("sharded", 2), ("sharded", 3)):
        a = out[(mode, world, 0)]
        for r in range(world):
            assert out[(mode, world, r)]["refused"] == (mode == "sharded"), (mode, world, r)
        for r in range(1, world):
            b = out[(mode, world, r)]
            # replicas bit-identical (parameters, gathered moments, statistics, step)
            assert a["checksum"] == b["checksum"], (mode, world)
            assert a["step"] == b["step"] == 3
            for f in FIELDS:
                assert np.array_equal(a["p"][f], b["p"][f]), (mode, world, f)
                assert np.array_equal(a["m"][f], b["m"][f]), (mode, world, f)
                assert np.array_equal(a["v"][f], b["v"][f]), (mode, world, f)
            for x, y in zip(a["stats"], b["stats"]):
                assert np.array_equal(x, y), (mode, world)
        if world == 2:
            # the first iteration: the ranks' one-view losses average to the
            # one-process 2-view loss
            b = out[(mode, world, 1)]
            assert (a["losses"][0] + b["losses"][0]) / 2 == pytest.approx(res["ref_loss"], rel=1e-6)
    # sharded (2 or 3 ranks; with 3, one rank renders no view) == all-reduce
    # exchange, up to K6's atomic summation order
    ar = out[("allreduce", 2, 0)]
    for world in (2, 3):
        sh = out[("sharded", world, 0)]
        for f in FIELDS:
            assert np.allclose(sh["p"][f], ar["p"][f], rtol=1e-5, atol=1e-7), (world, f)
            assert np.allclose(sh["m"][f], ar["m"][f], rtol=1e-4, atol=1e-9), (world, f)
            assert np.allclose(sh["v"][f], ar["v"][f], rtol=1e-4, atol=1e-12), (world, f)
        for x, y in zip(sh["stats"], ar["stats"]):
            assert np.allclose(x, y, rtol=1e-5, atol=1e-12), world
    # a non-finite loss on one rank: every rank aborts the same iteration,
    # keeps the previous parameters, and continues in lock step
    for mode in ("allreduce", "sharded"):
        r0, r1 = out[("abort", mode, 0)], out[("abort", mode, 1)]
        assert r0 == r1, mode
        assert [k for k, _ in r0] == ["ok", "abort", "ok"], (mode, r0)
        assert r0[1][1] == r0[0][1] and r0[2][1] != r0[1][1], mode
    # broadcast repair: rank 1 diverged, both end on rank 0's parameters
    b0, a0 = out[("allreduce", 2, 0, "repair")]
    b1, a1 = out[("allreduce", 2, 1, "repair")]
    assert b1 != b0 and a0 == a1 == b0
