"""Input pipeline host logic (no GPU): the dataset's epoch / batch semantics are the reference's
(dataset.py:93-142, pinned via oracle.ref_ops which tests/test_oracle_golden.py checks against the real
reference), and the crop/flip draw is the oracle's (restated.draw_crop_flip)."""

import numpy as np

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
