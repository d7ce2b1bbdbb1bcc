"""View-parallel exchange semantics on CPU (gloo, world_size 2).

The multi-GPU trainer (paper_2505_13215_b200/train.py) shards the batch by
view (rank r takes items b mod n == r), sums the per-view gradients already
scaled by 1/B plus the densification-statistic deltas with ONE all-reduce of a
packed buffer, then every rank applies the same Adam step.  This test runs that
protocol with the FP64 oracle as the per-view compute on two gloo ranks and
checks it against the single-process reference iteration (train.cpp:402-450):
same parameters, same statistics, bit-identical replicas.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

FIELDS = ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4", "mean3", "quat3", "log_s3", "op3", "sh3")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import oracle as O
    from paper_2505_13215_b200.train import quantize_8bit

    rng = O.Rng(5)
    scene = rng.random_scene(12, 12, 1)
    target = rng.random_scene(12, 12, 1)
    cams = [rng.random_camera(40, 32) for _ in range(4)]
    times = [0.2, 0.4, 0.6, 0.8]
    gts = [quantize_8bit(O.rasterize(target, c, t, (0.2, 0.2, 0.2))["rgb"]) for c, t in zip(cams, times)]
    return scene, cams, times, gts


def _worker(rank, world, port, q):
    import oracle as O
    from paper_2505_13215_b200.train import shard_batch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams, times, gts = _setup()
    st = O.AdamState(scene)
    batch = [0, 1, 2, 3]
    B = len(batch)
    acc = O.zero_grads(scene)
    dgn4, dgn3 = np.zeros(scene.n4), np.zeros(scene.n3)
    dc4, dc3 = np.zeros(scene.n4), np.zeros(scene.n3)
    loss = 0.0
    for v in shard_batch(batch, rank, world):
        img, tape = O.forward_train(scene, cams[v], times[v], (0.2, 0.2, 0.2))
        lv, lg = O.photometric_loss_with_grad(img, gts[v], 0.2)
        loss += lv
        g = O.backward(scene, cams[v], tape, lg)
        O.grads_add_scaled(scene, acc, g, 1.0 / B)
        dgn4 += np.where(g["screen_norm4"] > 0, g["screen_norm4"], 0.0)
        dc4 += g["screen_norm4"] > 0
        dgn3 += np.where(g["screen_norm3"] > 0, g["screen_norm3"], 0.0)
        dc3 += g["screen_norm3"] > 0
    # one packed all-reduce: gradients + statistic deltas + loss
    parts = [acc[f].ravel() for f in FIELDS] + [dgn4, dgn3, dc4, dc3, np.array([loss])]
    packed = torch.from_numpy(np.concatenate(parts))
    dist.all_reduce(packed)
    flat = packed.numpy()
    o = 0
    for f in FIELDS:
        n = acc[f].size
        acc[f] = flat[o:o + n].reshape(acc[f].shape).copy()
        o += n
    for arr in (dgn4, dgn3, dc4, dc3):
        arr[...] = flat[o:o + arr.size]
        o += arr.size
    loss = flat[o] / B
    st.grad_norm4 += dgn4
    st.grad_norm3 += dgn3
    st.count4 += dc4.astype(np.uint32)
    st.count3 += dc3.astype(np.uint32)
    O.optimizer_step(scene, acc, st)
    digest = np.concatenate([getattr(scene, f).ravel() for f in FIELDS])
    out = torch.from_numpy(digest)
    gathered = [torch.zeros_like(out) for _ in range(world)]
    dist.all_gather(gathered, out)
    if rank == 0:
        q.put({"params": {f: getattr(scene, f) for f in FIELDS}, "loss": loss,
               "gn4": st.grad_norm4.copy(), "c4": st.count4.copy(), "gn3": st.grad_norm3.copy(),
               "c3": st.count3.copy(), "replicas_equal": bool(torch.equal(gathered[0], gathered[1]))})
    dist.destroy_process_group()


def test_shard_batch_partitions():
    from paper_2505_13215_b200.train import shard_batch

    for world in (1, 2, 3, 4, 8):
        batch = list(range(13))
        shards = [shard_batch(batch, r, world) for r in range(world)]
        assert sorted(sum(shards, [])) == batch
        assert max(len(s) for s in shards) - min(len(s) for s in shards) <= 1


def test_view_parallel_step_matches_single_process():
    import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res["replicas_equal"]
    # single-process reference iteration over the same batch
    scene, cams, times, gts = _setup()
    st = O.AdamState(scene)
    loss = O.train_step(scene, st, cams, times, gts, (0.2, 0.2, 0.2), num_threads=1)
    assert res["loss"] == pytest.approx(loss, rel=1e-12)
    for f in FIELDS:
        np.testing.assert_allclose(res["params"][f], getattr(scene, f), rtol=1e-9, atol=1e-12, err_msg=f)
    np.testing.assert_allclose(res["gn4"], st.grad_norm4, rtol=1e-12)
    np.testing.assert_allclose(res["gn3"], st.grad_norm3, rtol=1e-12)
    assert (res["c4"] == st.count4).all() and (res["c3"] == st.count3).all()


def _abort_worker(rank, world, port, q):
    from paper_2505_13215_b200._capi import NumericAbort
    from paper_2505_13215_b200.train import reduce_batch_loss

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    out.append(reduce_batch_loss(dist, None, 0.25 + rank))            # finite on both ranks
    try:
        reduce_batch_loss(dist, None, float("nan") if rank == 1 else 0.5)
        out.append("no-abort")
    except NumericAbort:
        out.append("abort")
    out.append(reduce_batch_loss(dist, None, 1.0))                     # collectives still aligned
    dist.destroy_process_group()
    q.put((rank, out))


def test_numeric_abort_is_a_collective_decision():
    """One rank's non-finite view loss makes EVERY rank raise NumericAbort at
    the same step (the batch loss is all-reduced before the gradients)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_abort_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert res[r] == [1.5, "abort", 2.0], res


class _FakeReplica:
    """Stands in for a Context: a byte-string 'device state' that
    save_checkpoint / load_checkpoint move through files (as the real one)."""

    def __init__(self, state: bytes):
        self.state = state

    def param_checksum(self) -> int:
        import zlib

        return zlib.crc32(self.state)

    def save_checkpoint(self, path):
        with open(path, "wb") as f:
            f.write(self.state)

    def load_checkpoint(self, path):
        with open(path, "rb") as f:
            self.state = f.read()
        return True


def _replica_worker(rank, world, port, q):
    from paper_2505_13215_b200.train import repair_from_root, replicas_agree

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = _FakeReplica(b"scene-v1")
    out = [replicas_agree(dist, None, ctx.param_checksum())]          # identical replicas
    if rank == 1:
        ctx.state = b"scene-v1-diverged"
    ok = replicas_agree(dist, None, ctx.param_checksum())
    out.append(ok)
    if not ok:                                                        # every rank takes the same branch
        repair_from_root(dist, None, rank, ctx)
    out.append(ctx.state)
    out.append(replicas_agree(dist, None, ctx.param_checksum()))
    dist.destroy_process_group()
    q.put((rank, out))


def test_replica_check_and_repair():
    """ranks compare parameter checksums; a diverged replica is
    repaired from rank 0's checkpoint image, and all ranks decide together."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert res[r] == [True, False, b"scene-v1", True], res
