"""Input pipeline host logic (no GPU): the dataset's epoch / batch semantics are the reference's
(dataset.py:93-142, pinned via oracle.ref_ops which tests/test_oracle_golden.py checks against the real
reference), and the crop/flip draw is the oracle's (restated.draw_crop_flip)."""

import numpy as np
import pytest

from oracle import ref_ops as R
from oracle import restated as X


def test_dataset_epochs_match_reference_semantics():
    from paper_2409_11600_b200.data import ImageDataset

    n, b, seed = 53, 8, 5
    feats = np.arange(n * 3 * 2 * 2, dtype=np.float32).reshape(n, 3, 2, 2)
    ds = ImageDataset(feats, np.arange(n) % 10, b, seed=seed)
    perms = R.epoch_permutation(seed, n, 3)
    for e in range(3):
        ds.reset_epoch()
        np.testing.assert_array_equal(ds.permutation, perms[e])
        assert ds.num_batches() == 7
        got = np.concatenate([ds.batch_rows(i) for i in range(ds.num_batches())])
        np.testing.assert_array_equal(got, perms[e])  # exact coverage, partial last batch kept
        np.testing.assert_array_equal(ds.batch_rows(6), R.batch_rows(perms[e], 6, b))
    ds2 = ImageDataset(feats, np.zeros(n), b, seed=seed, shuffle=False)
    ds2.reset_epoch()
    np.testing.assert_array_equal(ds2.permutation, np.arange(n))


def test_crop_flip_draw_is_the_oracle_draw():
    from paper_2409_11600_b200.data import _draw_crop_flip, batch_generator

    for pad in (2, 4):
        a = _draw_crop_flip(batch_generator(3, 1, 7), 33, pad)
        b = X.draw_crop_flip(batch_generator(3, 1, 7), 33, pad)
        np.testing.assert_array_equal(a, b)
        assert a[:, :2].max() <= 2 * pad and a[:, 2].max() <= 1


def test_rank_shards_union_is_the_global_batch():
    """§8(e): every rank draws the same global permutation and takes its contiguous slice of each global batch;
    the union over ranks (in rank order) is the single-process batch, bit for bit."""
    from paper_2409_11600_b200.data import ImageDataset

    n, b, seed = 96, 16, 3
    feats = np.zeros((n, 3, 2, 2), np.float32)
    single = ImageDataset(feats, np.arange(n) % 10, b, seed=seed)
    for world in (2, 4):
        shards = [ImageDataset(feats, np.arange(n) % 10, b, seed=seed, rank=r, world=world) for r in range(world)]
        for e in range(2):
            single.reset_epoch() if world == 2 else None
            for ds in shards:
                ds.reset_epoch()
            if world == 4:  # single-process reference for the same epoch
                ref = ImageDataset(feats, np.arange(n) % 10, b, seed=seed)
                for _ in range(e + 1):
                    ref.reset_epoch()
            else:
                ref = single
            for i in range(ref.num_batches()):
                parts = [ds.batch_rows(i) for ds in shards]
                assert all(len(p) == b // world for p in parts)
                np.testing.assert_array_equal(np.concatenate(parts), ref.batch_rows(i))


def test_rank_shard_rejects_uneven_split():
    import pytest

    from paper_2409_11600_b200.data import ImageDataset
    from paper_2409_11600_b200.errors import NskRuntimeError

    with pytest.raises(NskRuntimeError):
        ImageDataset(np.zeros((8, 1), np.float32), np.zeros(8), 6, rank=0, world=4)


class _FakeSlot:
    """Host-only stand-in for data.PinnedSlot (no pinned memory, no CUDA event)."""

    def __init__(self, b):
        self.arrays = {"x": np.zeros((b, 1), np.float32), "y": np.zeros(b, np.float32)}
        self.index, self.rows = -1, 0

    def wait_copied(self):
        pass


def _host_loader(n, b, workers, capacity):
    """A DeviceLoader without device resources: the producer/consumer logic is host-only."""
    import queue

    from paper_2409_11600_b200.data import DeviceLoader, ImageDataset

    ds = ImageDataset(np.arange(n, dtype=np.float32).reshape(n, 1), np.arange(n) % 10, b, seed=1)
    ld = DeviceLoader.__new__(DeviceLoader)
    ld.ds, ld.workers, ld.capacity, ld.pad = ds, workers, capacity, 0
    ld.slots = [_FakeSlot(b) for _ in range(capacity + 1)]
    ld._free = queue.Queue()
    for sl in ld.slots:
        ld._free.put(sl)
    ld._epoch, ld._threads, ld._cursor = None, [], 0
    return ld


def _drain(ld, limit=None):
    from paper_2409_11600_b200.data import END_OF_DATA

    got = []
    while limit is None or len(got) < limit:
        sl = ld._next_slot()
        if sl is END_OF_DATA:
            break
        got.append((sl.index, sl.arrays["x"][:sl.rows, 0].astype(np.int64).copy()))
        ld._free.put(sl)  # what next() does once the copy is issued
    return got


def test_reset_epoch_mid_epoch_with_full_ring_does_not_deadlock():
    """reset_epoch with workers blocked on a full ring must stop them, return every staged slot and
    start a clean epoch (the reference builds a fresh queue per epoch, dataset.py:103-109)."""
    import threading
    import time

    n, b, workers, cap = 200, 8, 3, 2
    ld = _host_loader(n, b, workers, cap)
    ld.reset_epoch()
    _drain(ld, limit=2)
    time.sleep(0.2)  # workers fill the ring and block
    done = threading.Event()

    def reset_and_read():
        ld.reset_epoch()
        done.result = _drain(ld)
        done.set()

    th = threading.Thread(target=reset_and_read, daemon=True)
    th.start()
    assert done.wait(20), "reset_epoch mid-epoch deadlocked"
    got = done.result
    assert sorted(i for i, _ in got) == list(range(ld.ds.num_batches()))
    rows = np.sort(np.concatenate([r for _, r in got]))
    np.testing.assert_array_equal(rows, np.arange(n))  # exact coverage of the NEW epoch's permutation
    for i, r in got:
        np.testing.assert_array_equal(r, ld.ds.batch_rows(i))
    ld.shutdown()
    assert ld._free.qsize() == len(ld.slots)  # every slot back in the ring


def test_cifar_binary_round_trip(tmp_path):
    """On-disk format: CIFAR-10 binary records (label byte + R, G, B planes) read as uint8
    NHWC images bit-exactly, files concatenated in order; malformed sizes raise the reference's runtime error."""
    from paper_2409_11600_b200 import data
    from paper_2409_11600_b200.errors import NskRuntimeError

    rng = np.random.default_rng(3)
    im1 = rng.integers(0, 256, (5, 32, 32, 3), dtype=np.uint8)
    im2 = rng.integers(0, 256, (3, 32, 32, 3), dtype=np.uint8)
    lb1, lb2 = rng.integers(0, 10, 5), rng.integers(0, 10, 3)
    p1, p2 = tmp_path / "data_batch_1.bin", tmp_path / "data_batch_2.bin"
    data.write_cifar_bin(p1, im1, lb1)
    data.write_cifar_bin(p2, im2, lb2)
    assert p1.stat().st_size == 5 * data.CIFAR_RECORD
    raw = np.fromfile(p1, np.uint8).reshape(5, -1)  # the published layout: label, then the red plane row-major
    assert raw[2, 0] == lb1[2] and raw[2, 1 + 7 * 32 + 9] == im1[2, 7, 9, 0] and raw[2, 1 + 1024 + 5] == im1[2, 0, 5, 1]
    x, y = data.read_cifar_bin([p1, p2])
    assert x.dtype == np.uint8 and x.shape == (8, 32, 32, 3) and x.flags["C_CONTIGUOUS"]
    np.testing.assert_array_equal(x, np.concatenate([im1, im2]))
    np.testing.assert_array_equal(y, np.concatenate([lb1, lb2]).astype(np.float32))
    ds = data.ImageDataset.from_cifar_bin(str(p1), batch_size=2, seed=1)
    assert ds.uint8 and ds.num_rows == 5 and ds.num_batches() == 3
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\0" * (data.CIFAR_RECORD + 1))
    with pytest.raises(NskRuntimeError):
        data.read_cifar_bin(bad)
