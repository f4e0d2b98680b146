"""Data parallelism executed: the product DataParallel -- bucket layout, param-fire hooks,
comm stream, 1/N folded into the optimizer -- run for real.

* one rank over a real NCCL communicator inside a CUDA-graph-captured step: bit-identical to the same step without
  data parallelism (the all-reduce of one rank is the identity; ordering and capture must not change anything);
* two processes sharing the GPU, each training on its rank's shard of the same global batch (ImageDataset with
  rank/world), with the bucket all-reduce carried by a host gloo process group instead of NCCL (NCCL refuses two
  ranks on one device): the averaged gradients and the SGD update equal the single-process full-batch oracle.
"""

import ctypes as C
import os
import socket

import numpy as np
import pytest

from oracle import models as om

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_dp_one_rank_nccl_captured_step_is_bit_identical(dev):
    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200.dp import DataParallel
    from paper_2409_11600_b200.models import ResNet18
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(5)
    xs = [rng.standard_normal((32, 3, 32, 32)).astype(np.float32) for _ in range(5)]
    ys = [rng.integers(0, 10, 32).astype(np.float32) for _ in range(5)]
    runs = {}
    for use_dp in (False, True):
        s = Session(seed=0)
        net = ResNet18(s)
        dp = None
        if use_dp:
            raw = (C.c_uint8 * 128)()
            _lib.check(_lib.lib().nsk_comm_unique_id(raw))
            dp = DataParallel(s, 0, 1, bucket_mb=1.0, uid=bytes(raw))
        tr = Trainer(s, net, xs[0].shape, 10, optimizer=("sgd", 0.05, 0.9), graph=True, warmup=2, dp=dp)
        losses = [float(tr.step(x, y)) for x, y in zip(xs, ys)]
        assert tr.graph is not None  # steps 3.. replayed a captured graph (with the NCCL calls inside)
        runs[use_dp] = (losses, {n: t.data.copy() for n, t in s.param_group.params}, dp)
    assert runs[True][0] == runs[False][0]
    for n in runs[False][1]:
        np.testing.assert_array_equal(runs[True][1][n], runs[False][1][n])
    dp = runs[True][2]
    assert dp.buckets is not None and len(dp.buckets) > 1
    # every bucket launched once per bucketed step, from the param-fire hook (reverse declaration order first)
    nb = len(dp.buckets)
    assert sorted(dp.launch_log[:nb]) == list(range(nb))


def test_dp_one_rank_nccl_adamw_clip_gru_step_is_bit_identical(dev):
    """The AdamW + clip_grad_norm path under data parallelism (gradients scaled by 1/N before the norm is taken,
    the update without the group scale) on the C3 model family through the tcgen05 GRU: one NCCL rank inside a
    captured step equals the step without data parallelism bit for bit."""
    from paper_2409_11600_b200 import _lib, nn
    from paper_2409_11600_b200.dp import DataParallel
    from paper_2409_11600_b200.models import GRUClassifier
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(6)
    V, T, B = 1000, 16, 16
    xs = [rng.integers(0, V, (B, T)).astype(np.float32) for _ in range(5)]
    ys = [rng.integers(0, 2, B).astype(np.float32) for _ in range(5)]
    runs = {}
    for use_dp in (False, True):
        s = Session(seed=0)
        model = GRUClassifier(s, vocab=V, embed=128, hidden=128)
        dp = None
        if use_dp:
            raw = (C.c_uint8 * 128)()
            _lib.check(_lib.lib().nsk_comm_unique_id(raw))
            dp = DataParallel(s, 0, 1, bucket_mb=1.0, uid=bytes(raw))
        opt = ("adamw", nn.Hyperparams(learning_rate=1e-3, weight_decay=1e-4), 0.5)  # the clip engages
        tr = Trainer(s, model, (B, T), 2, optimizer=opt, graph=True, warmup=2, dp=dp)
        losses = [float(tr.step(x, y)) for x, y in zip(xs, ys)]
        assert tr.graph is not None
        runs[use_dp] = (losses, {n: t.data.copy() for n, t in s.param_group.params})
    assert runs[True][0] == runs[False][0]
    for n in runs[False][1]:
        np.testing.assert_array_equal(runs[True][1][n], runs[False][1][n])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORLD, GLOBAL_B, ROWS = 2, 32, 64


def _dataset():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((ROWS, 3, 16, 16)).astype(np.float32)
    y = rng.integers(0, 10, ROWS).astype(np.float32)
    return x, y


def _dp_worker(rank, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200.data import ImageDataset
    from paper_2409_11600_b200.dp import DataParallel
    from paper_2409_11600_b200.models import SmallCNN
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    _lib.ctx.init(0)
    lib = _lib.lib()

    def host_allreduce(ptr, count, dtype, stream):
        assert dtype == _lib.F32
        _lib.check(lib.nsk_stream_sync(stream))
        arr = np.empty(count, np.float32)
        _lib.check(lib.nsk_memcpy_d2h(arr.ctypes.data, ptr, 4 * count, stream))
        _lib.check(lib.nsk_stream_sync(stream))
        t = torch.from_numpy(arr)
        dist.all_reduce(t)
        _lib.check(lib.nsk_memcpy_h2d(ptr, arr.ctypes.data, 4 * count, stream))
        _lib.check(lib.nsk_stream_sync(stream))

    try:
        x, y = _dataset()
        ds = ImageDataset(x, y, GLOBAL_B, seed=4, rank=rank, world=WORLD)
        ds.reset_epoch()
        s = Session(seed=0)
        net = SmallCNN(s, hw=16)
        dp = DataParallel(s, rank, WORLD, bucket_mb=0.02, allreduce=host_allreduce)
        tr = Trainer(s, net, (GLOBAL_B // WORLD, 3, 16, 16), 10, optimizer=("sgd", 0.01, 0.9), graph=False, dp=dp)
        grads, params = [], []
        for i in range(2):
            rows = ds.batch_rows(i)
            # capture the all-reduced (summed) gradients before the optimizer consumes and zeroes them
            orig = dp.finish_backward

            def finish_and_record(orig=orig):
                orig()
                _lib.sync()
                grads.append({n: s.grad_cache.get(n).copy() for n, _t in s.param_group.params})

            dp.finish_backward = finish_and_record
            float(tr.step(x[rows], y[rows]))
            dp.finish_backward = orig
            params.append({n: t.data.copy() for n, t in s.param_group.params})
        correct = dp.allreduce_count(rank + 1)
        out_q.put((rank, grads, params, dp.buckets is not None and len(dp.buckets), list(dp.launch_log), correct))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_dp_two_processes_bucketed_allreduce_matches_full_batch_oracle(dev):
    import torch.multiprocessing as mp

    from paper_2409_11600_b200.data import ImageDataset

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        r = q.get(timeout=600)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, y = _dataset()
    ds = ImageDataset(x, y, GLOBAL_B, seed=4)
    ds.reset_epoch()
    ref = om.SmallCNNOracle(seed=0, hw=16)
    names = ["w1", "b1", "w2", "b2", "fc_w", "fc_b"]
    g0, p0, nbuckets, log0, correct = res[0]
    g1, p1, _, _, _ = res[1]
    assert correct == 3  # integer sum over ranks (accuracy counts)
    assert nbuckets and nbuckets > 1
    assert sorted(log0[:nbuckets]) == list(range(nbuckets))  # step 2: every bucket launched from its hook
    pnames = sorted(g0[0], key=lambda n: int(n[1:]))
    dev_prev = {pn: ref.params[key].copy() for pn, key in zip(pnames, names)}  # bit-identical init
    for i in range(2):
        rows = ds.batch_rows(i)
        _loss, gref, _ = ref.loss_and_grads(x[rows], y[rows], bf16=True)
        ref_prev = {k: v.copy() for k, v in ref.params.items()}
        ref.opt.sgd(ref.params, gref, 0.01, 0.9)
        for pname, key in zip(pnames, names):
            np.testing.assert_array_equal(g0[i][pname], g1[i][pname])  # both ranks hold the same reduced sum
            avg = g0[i][pname] / WORLD
            assert _rel(avg, gref[key]) < 1e-3, (i, key, _rel(avg, gref[key]))
            np.testing.assert_array_equal(p0[i][pname], p1[i][pname])  # replicas stay identical
            upd = dev_prev[pname].astype(np.float64) - p0[i][pname]  # the applied SGD update (1/N folded in)
            ref_upd = ref_prev[key].astype(np.float64) - ref.params[key]
            assert _rel(upd, ref_upd) < 1e-3, (i, key, _rel(upd, ref_upd))
            dev_prev[pname] = p0[i][pname]
