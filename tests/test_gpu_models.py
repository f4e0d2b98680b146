"""Whole-step parity: device training steps vs the CPU oracle on identical seeds and inputs."""

import numpy as np
import pytest

from oracle import models as om

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_small_cnn_one_sgd_step_matches_oracle(session):
    """C1: small CNN, one SGD step; loss and every updated parameter vs the bf16-emulating oracle."""
    from paper_2409_11600_b200.models import SmallCNN
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(0)
    x = rng.standard_normal((32, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, 32).astype(np.float32)
    model = SmallCNN(session)
    w0 = {n: t.data.copy() for n, t in session.param_group.params}
    tr = Trainer(session, model, x.shape, 10, optimizer=("sgd", 0.01, 0.9), graph=False)
    loss = float(tr.step(x, y))
    ref = om.SmallCNNOracle(seed=0)
    names = ["w1", "b1", "w2", "b2", "fc_w", "fc_b"]
    for (n, _t), key in zip(session.param_group.params, names):
        np.testing.assert_array_equal(w0[n], ref.params[key])  # bit-identical init (seed plumbing)
    ref_loss = ref.train_step(x, y, lr=0.01, momentum=0.9, bf16=True)
    assert abs(loss - ref_loss) <= 1e-3 * abs(ref_loss)
    for (pname, t), key in zip(session.param_group.params, names):
        # the applied update (w0 - w1)/lr is the gradient: within 1% (bf16 storage on both sides)
        upd = (w0[pname].astype(np.float64) - t.data) / 0.01
        ref_upd = (w0[pname].astype(np.float64) - ref.params[key]) / 0.01
        assert _rel(upd, ref_upd) < 1e-2, (pname, key, _rel(upd, ref_upd))


def test_resnet18_gradients_match_oracle(session):
    """C2 at a small batch: loss, logits and every parameter gradient of one forward/backward."""
    from paper_2409_11600_b200 import autodiff, nn
    from paper_2409_11600_b200.models import ResNet18

    rng = np.random.default_rng(1)
    b = 8
    x = rng.standard_normal((b, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, b).astype(np.float32)
    model = ResNet18(session)
    assert model.num_params() == 11_173_962
    ref = om.ResNet18Oracle(seed=0)
    for (n, t), key in zip(session.param_group.params, ref.order):
        np.testing.assert_array_equal(t.data, ref.params[key])  # bit-identical init (seed plumbing)
    pool = session.pool
    logits = model.forward(autodiff.make_data(pool, x))
    dlogits = logits.data
    loss = nn.cross_entropy(logits, autodiff.make_data(pool, y), pool)
    session.push_named("loss", loss)
    autodiff.backward(session.tape(), session.grad_cache, pool)
    ref_loss, grads, ref_logits = ref.loss_and_grads(x, y, bf16=True)
    assert _rel(dlogits, ref_logits) < 3e-2  # near-zero logits at init: bf16 activations dominate
    assert abs(loss.item() - ref_loss) <= 2e-3 * abs(ref_loss), (loss.item(), ref_loss)
    # At initialisation early-layer gradients are ill-conditioned w.r.t. the forward activations: rounding
    # only the oracle's forward activations to bf16 (backward exact) already moves them by ~37% vs float64
    # ("parity"). Per-op parity is held at 1e-3 in test_gpu_ops.py; here the head of the network
    # must agree tightly and every gradient must point the same way.
    pairs = [(n, key) for (n, _t), key in zip(session.param_group.params, ref.order)]
    for n, key in pairs:
        g = session.grad_cache.get(n).astype(np.float64).ravel()
        r = grads[key].astype(np.float64).ravel()
        cos = float(g @ r / (np.linalg.norm(g) * np.linalg.norm(r) + 1e-30))
        assert cos > 0.9, (key, cos)
        if key.startswith("fc_"):
            assert _rel(g, r) < 2e-2, (key, _rel(g, r))


def test_resnet18_graph_replay_matches_eager(dev):
    """Captured-and-replayed steps produce the same losses as eager steps."""
    from paper_2409_11600_b200.models import ResNet18
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(2)
    b = 16
    xs = [rng.standard_normal((b, 3, 32, 32)).astype(np.float32) for _ in range(5)]
    ys = [rng.integers(0, 10, b).astype(np.float32) for _ in range(5)]
    losses = {}
    for mode in (False, True):
        s = Session(seed=0)
        tr = Trainer(s, ResNet18(s), xs[0].shape, 10, optimizer=("sgd", 0.1, 0.9), graph=mode, warmup=2)
        losses[mode] = [float(tr.step(x, y)) for x, y in zip(xs, ys)]
        if mode:
            assert tr.graph is not None and tr.launches_per_step > 100
    np.testing.assert_allclose(losses[True], losses[False], rtol=1e-5)
