"""Host-side logic that needs no GPU: Pool semantics, tape bookkeeping, DP buckets (reference test_tensor.py:35-119).

The Pool's device allocations are replaced by a host stub so its free-list contract (exact-size
keys, LIFO, no zeroing, disabled baseline, double-release guard, conservation) is checked here;
the GPU suite exercises the same Pool over real HBM.
"""

import random

import pytest

from paper_2409_11600_b200 import tensor as T
from paper_2409_11600_b200.errors import NskRuntimeError


class FakeBuffer:
    def __init__(self, capacity, dtype=0, base=None, offset=0):
        self.capacity, self.dtype, self.origin, self.in_pool, self.base = capacity, dtype, "fresh", False, base
        self.ptr = id(self)
        self.freed = False

    def fill(self, v):
        self.filled = v

    def free(self):
        self.freed = True


@pytest.fixture(autouse=True)
def fake_buffers(monkeypatch):
    monkeypatch.setattr(T, "Buffer", FakeBuffer)


def test_first_acquire_is_fresh():
    pool = T.Pool()
    buf = pool.acquire(512)
    assert buf.origin == "fresh"
    assert pool.stats() == {"fresh": 1, "hits": 0, "released": 0}


def test_release_then_acquire_returns_same_buffer():
    pool = T.Pool()
    buf = pool.acquire(512)
    pool.release(buf)
    again = pool.acquire(512)
    assert again is buf and again.origin == "pooled" and pool.stats()["hits"] == 1


def test_exact_size_and_dtype_keying():
    pool = T.Pool()
    buf = pool.acquire(512)
    pool.release(buf)
    assert pool.acquire(256) is not buf
    assert pool.acquire(512, dtype=1) is not buf  # bf16 buffers live in their own free lists
    assert pool.stats()["fresh"] == 3


def test_lifo_reuse_order():
    pool = T.Pool()
    a, b = pool.acquire(64), pool.acquire(64)
    pool.release(a)
    pool.release(b)
    assert pool.acquire(64) is b and pool.acquire(64) is a


def test_double_release_rejected():
    pool = T.Pool()
    buf = pool.acquire(8)
    pool.release(buf)
    with pytest.raises(NskRuntimeError):
        pool.release(buf)


def test_poison_fills_nan_and_disabled_pool_frees():
    pool = T.Pool(poison=True)
    b = pool.acquire(4)
    pool.release(b)
    assert b.filled != b.filled  # NaN
    off = T.Pool(enabled=False)
    a = off.acquire(32)
    off.release(a)
    assert a.freed and off.acquire(32) is not a and off.stats()["fresh"] == 2


def test_invalid_size():
    with pytest.raises(NskRuntimeError):
        T.Pool().acquire(0)


def test_pool_conservation_random_sequence():
    rng = random.Random(7)
    pool = T.Pool()
    live = []
    for _ in range(500):
        if live and rng.random() < 0.5:
            pool.release(live.pop(rng.randrange(len(live))))
        else:
            live.append(pool.acquire(rng.choice([16, 32, 64])))
        s = pool.stats()
        assert s["fresh"] + s["hits"] == s["released"] + len(live)
        assert pool.free_total() == s["released"] - s["hits"]


def test_tape_recording_structure():
    """Tree shape of x@w + x and consumer counts (test_autodiff.py:17-28) without device math."""
    from paper_2409_11600_b200 import autodiff as ad

    pool = T.Pool()
    x = T.Tensor((1, 1), pool.acquire(1), param_name="x")
    w = T.Tensor((1, 1), pool.acquire(1), param_name="w")
    h = T.Tensor((1, 1), pool.acquire(1))
    ad.record("matmul_t", h, x, w, saved=(x, w))
    y = T.Tensor((1, 1), pool.acquire(1))
    root = ad.record("add", y, h, x)
    assert root.op == "add" and root.left.op == "matmul_t"
    assert root.left.left.op == "param" and root.left.left.param_name == "x"
    assert root.right is root.left.left
    assert root.left.left.consumers == 2 and x.refs == 1 and w.refs == 1
    tape = ad.Tape()
    ad.push_assignment(tape, "s.y", y)
    assert root.pushed and root.consumers == 1 and [k for k, _ in tape.entries] == ["s.y"]
    tape.sealed = True
    with pytest.raises(NskRuntimeError, match="sealed"):
        ad.push_assignment(tape, "s.z", h)


def test_dp_bucket_layout():
    """Buckets are contiguous slices of the flat grad arena, filled in reverse declaration order."""
    from paper_2409_11600_b200.dp import DataParallel

    class Cache:
        pass

    cache = Cache()
    sizes = {"p0": 1000, "p1": 3000, "p2": 500, "p3": 6000}
    offs, total = {}, 0
    for name in reversed(list(sizes)):
        offs[name] = total
        total += (sizes[name] + 7) // 8 * 8
    cache.offsets = offs
    cache.grads = {n: FakeBuffer(s) for n, s in sizes.items()}
    cache.arena = FakeBuffer(total)
    dp = DataParallel.__new__(DataParallel)
    dp.bucket_elems = 5000

    class S:
        grad_cache = cache

    dp.s = S()
    import paper_2409_11600_b200.dp as dpmod

    dpmod._event = lambda: 0
    dp._build_buckets()
    covered = sorted((s, s + c) for s, c, _ in dp.buckets)
    assert covered[0][0] == 0 and covered[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
    assert dp.buckets[0][2][0] == "p3"  # last declared parameter finishes first in backward
    assert set(dp.owner) == set(sizes)
