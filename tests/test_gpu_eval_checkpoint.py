"""§8(f) 4: eval mode (BatchNorm running statistics) and checkpoint save/restore of the training state."""

import numpy as np
import pytest

from oracle import restated as X

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_batchnorm_running_stats_and_eval_mode(session):
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    rng = np.random.default_rng(11)
    pool = session.pool
    c = 64
    gb = np.stack([rng.uniform(0.5, 1.5, c), rng.uniform(-0.5, 0.5, c)]).astype(np.float32)
    gbt = autodiff.make_param(pool, gb, "gb")
    rm, rv = np.zeros(c), np.ones(c)
    for step in range(3):
        x = X.round_bf16(rng.standard_normal((4, 8, 8, c)) * (1 + step) + step)
        layers.batchnorm(autodiff.make_data(pool, x, dtype=BF16), gbt, pool, relu=True)
        flat = x.reshape(-1, c).astype(np.float64)
        rm = 0.9 * rm + 0.1 * flat.mean(axis=0)
        rv = 0.9 * rv + 0.1 * flat.var(axis=0, ddof=1)
    run = layers.bn_running(gbt).host().reshape(2, c)
    np.testing.assert_allclose(run[0], rm, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(run[1], rv, rtol=1e-4)
    x = X.round_bf16(rng.standard_normal((4, 8, 8, c)))
    res = X.round_bf16(rng.standard_normal((4, 8, 8, c)))
    y = layers.batchnorm(autodiff.make_data(pool, x, dtype=BF16), gbt, pool, relu=True,
                         residual=autodiff.make_data(pool, res, dtype=BF16), training=False)
    scale = gb[0] / np.sqrt(run[1].astype(np.float64) + 1e-5)
    ref = np.maximum(x * scale + (gb[1] - run[0] * scale) + res, 0)
    assert rel(y.data, X.round_bf16(ref)) < 1e-3
    np.testing.assert_array_equal(layers.bn_running(gbt).host().reshape(2, c), run)  # eval does not update


def _resnet_trainer(graph=True):
    from paper_2409_11600_b200.models import ResNet18
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    s = Session(seed=0)
    return s, Trainer(s, ResNet18(s), (16, 3, 32, 32), 10, optimizer=("sgd", 0.05, 0.9), graph=graph, warmup=2)


def test_checkpoint_restores_training_bit_for_bit(dev, tmp_path):
    from paper_2409_11600_b200 import checkpoint

    rng = np.random.default_rng(12)
    xs = [rng.standard_normal((16, 3, 32, 32)).astype(np.float32) for _ in range(7)]
    ys = [rng.integers(0, 10, 16).astype(np.float32) for _ in range(7)]
    s, tr = _resnet_trainer()
    for x, y in zip(xs[:4], ys[:4]):
        float(tr.step(x, y))
    path = str(tmp_path / "ckpt.npz")
    checkpoint.save(s, path)
    assert int(np.load(path)["meta/step_count"][0]) == 4  # eager + captured + replayed SGD steps all counted
    cont = [float(tr.step(x, y)) for x, y in zip(xs[4:], ys[4:])]
    eval_a = tr.evaluate(xs[0], ys[0])
    s2, tr2 = _resnet_trainer()
    # a fresh model, optimizer and graph: warm it up on other data, then restore
    for x, y in zip(xs[:2], ys[:2]):
        float(tr2.step(x * 0.5, y))
    checkpoint.load(s2, path)
    resumed = [float(tr2.step(x, y)) for x, y in zip(xs[4:], ys[4:])]
    assert resumed == cont, (resumed, cont)
    assert s2.param_group.step_count == s.param_group.step_count == 7
    eval_b = tr2.evaluate(xs[0], ys[0])
    assert eval_a == eval_b


def test_evaluate_is_side_effect_free(dev):
    from paper_2409_11600_b200 import layers

    rng = np.random.default_rng(13)
    s, tr = _resnet_trainer()
    x = rng.standard_normal((16, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, 16).astype(np.float32)
    for _ in range(3):
        float(tr.step(x, y))
    params = {n: t.data.copy() for n, t in s.param_group.params}
    running = {n: layers.bn_running(t).host().copy() for n, t in s.param_group.params if t.shape[0] == 2
               and t in layers._RUNNING}
    a = tr.evaluate(x, y)
    b = tr.evaluate(x, y)
    assert a == b and np.isfinite(a[0]) and 0 <= a[1] <= 16
    for n, t in s.param_group.params:
        np.testing.assert_array_equal(t.data, params[n])
    for n, t in s.param_group.params:
        if n in running:
            np.testing.assert_array_equal(layers.bn_running(t).host(), running[n])
    after = float(tr.step(x, y))  # training continues (graph replay unaffected by the eval pass)
    assert np.isfinite(after)
