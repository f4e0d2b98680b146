"""Prefetching pinned-ring loader + GPU crop/flip on B200 vs the reference semantics and the oracle."""

import numpy as np
import pytest

from oracle import models as om
from oracle import restated as X

pytestmark = pytest.mark.gpu

MEAN, STD = (0.49, 0.48, 0.45), (0.25, 0.24, 0.26)


def _u8_dataset(n=64, hw=32, seed=9):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, (n, hw, hw, 3), dtype=np.uint8), rng.integers(0, 10, n).astype(np.float32)


def _trainer(b, graph=False):
    from paper_2409_11600_b200.models import ResNet18
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    s = Session(seed=0)
    return Trainer(s, ResNet18(s), (b, 32, 32, 3), 10, optimizer=("sgd", 0.1, 0.9), graph=graph, warmup=2,
                   augment=(4, MEAN, STD))


@pytest.mark.parametrize("workers", [1, 3])
def test_loader_delivers_each_batch_once_bit_exact(dev, workers):
    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200.data import END_OF_DATA, DeviceLoader, ImageDataset, _draw_crop_flip, batch_generator

    imgs, labels = _u8_dataset()
    ds = ImageDataset(imgs, labels, 16, seed=2)
    tr = _trainer(16)
    ld = DeviceLoader(ds, tr, workers=workers)
    for epoch in (1, 2):
        ld.reset_epoch()
        seen = []
        while True:
            idx = ld.next()
            if idx is END_OF_DATA:
                break
            _lib.sync()
            rows = ds.batch_rows(idx)
            raw = tr.x_dev.buffer.host().view(np.uint8)[: imgs[rows].size].reshape(imgs[rows].shape)
            np.testing.assert_array_equal(raw, imgs[rows])
            np.testing.assert_array_equal(tr.y_dev.buffer.host(), labels[rows])
            offs = tr.offs_dev.buffer.host().view(np.int32).reshape(-1, 3)
            np.testing.assert_array_equal(offs, _draw_crop_flip(batch_generator(2, epoch, idx), 16, 4))
            seen.append(idx)
        assert sorted(seen) == list(range(4))
        if workers == 1:
            assert seen == list(range(4))
        assert ld.next() is END_OF_DATA  # sticky
    ld.shutdown()


def test_augmented_step_matches_oracle(dev):
    """GPU crop/flip/normalise -> ResNet-18 step vs the oracle fed the restated augmentation."""
    imgs, labels = _u8_dataset(16)
    tr = _trainer(16)
    offs = X.draw_crop_flip(np.random.default_rng(4), 16, 4)
    loss = float(tr.step(imgs, labels, offsets=offs))
    aug = X.augment_crop_flip(imgs, offs, 4, MEAN, STD)  # NHWC float64
    ref = om.ResNet18Oracle(seed=0)
    ref_loss = ref.train_step(np.transpose(aug, (0, 3, 1, 2)), labels, lr=0.1, momentum=0.9, bf16=True)
    assert abs(loss - ref_loss) <= 2e-3 * abs(ref_loss), (loss, ref_loss)


def test_loader_fed_graph_replay_matches_eager(dev):
    """In-order loading (W=1): loader-fed captured steps reproduce eager steps; W=3 trains through the same
    graph with unordered delivery (concurrency.py semantics)."""
    from paper_2409_11600_b200.data import DeviceLoader, ImageDataset

    imgs, labels = _u8_dataset(96)
    out = {}
    for graph, workers in ((False, 1), (True, 1), (True, 3)):
        ds = ImageDataset(imgs, labels, 16, seed=1)
        tr = _trainer(16, graph=graph)
        ld = DeviceLoader(ds, tr, workers=workers)
        ld.reset_epoch()
        out[(graph, workers)] = [float(tr.run_staged()) for _ in range(ds.num_batches()) if ld.next() is not None]
        ld.shutdown()
    np.testing.assert_allclose(out[(True, 1)], out[(False, 1)], rtol=1e-5)
    assert len(out[(True, 3)]) == 6 and all(np.isfinite(out[(True, 3)]))


def test_cifar_binary_file_feeds_the_loader(dev, tmp_path):
    """CIFAR-10 binary batches on disk -> ImageDataset.from_cifar_bin -> pinned-ring loader -> GPU crop/flip ->
    graphed ResNet-18 steps: the staged batch is the file's bytes, and training runs through it."""
    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200.data import END_OF_DATA, DeviceLoader, ImageDataset, write_cifar_bin

    imgs, labels = _u8_dataset(48)
    write_cifar_bin(tmp_path / "data_batch_1.bin", imgs[:32], labels[:32])
    write_cifar_bin(tmp_path / "data_batch_2.bin", imgs[32:], labels[32:])
    ds = ImageDataset.from_cifar_bin([tmp_path / "data_batch_1.bin", tmp_path / "data_batch_2.bin"], 16, seed=4)
    tr = _trainer(16, graph=True)
    ld = DeviceLoader(ds, tr, workers=2)
    ld.reset_epoch()
    losses = []
    for _ in range(ds.num_batches()):
        idx = ld.next()
        if idx is END_OF_DATA:
            break
        _lib.sync()
        rows = ds.batch_rows(idx)
        raw = tr.x_dev.buffer.host().view(np.uint8)[: imgs[rows].size].reshape(imgs[rows].shape)
        np.testing.assert_array_equal(raw, imgs[rows])
        losses.append(float(tr.run_staged()))
    ld.shutdown()
    assert len(losses) == 3 and all(np.isfinite(losses))
