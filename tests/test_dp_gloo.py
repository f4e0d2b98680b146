"""Data-parallel semantics on CPU with two gloo ranks.

Each rank takes its contiguous slice of the same global batch (same seeded permutation on every
rank), computes its local gradient with the oracle, and the sum-all-reduce scaled by 1/N (what
the device path folds into the optimizer) must equal the single-process full-batch gradient.
The CE loss averages over the local rows inside its rule (autodiff.py:291), so equal shards make
the average of local means the global mean. The accuracy count is summed as an integer (bit-exact).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import models as om
from oracle import ref_ops as R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((16, 3, 16, 16)).astype(np.float32)
    y = rng.integers(0, 10, 16).astype(np.float32)
    perm = R.epoch_permutation(5, 16, 1)[0]  # identical on every rank
    b = 16 // world
    rows = perm[rank * b:(rank + 1) * b]
    model = om.SmallCNNOracle(seed=0, hw=16)
    _loss, grads, logits = model.loss_and_grads(x[rows], y[rows])
    red = {}
    for k in sorted(grads):
        t = torch.tensor(np.asarray(grads[k], np.float64))
        dist.all_reduce(t)
        red[k] = (t / world).numpy()
    correct = torch.tensor([int((logits.argmax(axis=1) == y[rows].astype(np.int64)).sum())])
    dist.all_reduce(correct)
    if rank == 0:
        out_q.put((red, int(correct[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gradient_average_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    red, correct = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    x = rng.standard_normal((16, 3, 16, 16)).astype(np.float32)
    y = rng.integers(0, 10, 16).astype(np.float32)
    model = om.SmallCNNOracle(seed=0, hw=16)
    _loss, full, logits = model.loss_and_grads(x, y)
    for k in full:
        np.testing.assert_allclose(red[k], full[k], rtol=1e-9, atol=1e-12)
    assert correct == int((logits.argmax(axis=1) == y.astype(np.int64)).sum())
