"""C3: fused GRU classifier (embedding -> GRU -> head -> CE) vs the float64 oracle composed from reference primitives."""

import numpy as np
import pytest

from oracle import models as om
from oracle import restated as X

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# (V, E, H, T, B): the first shape runs the fp32 cooperative recurrence (H = 64 is below the cluster kernel's
# tiling), the others the tcgen05 cluster kernel (gru_tc.cu); the last is configuration C3 itself
# (V, E, H, T, B): H = 64 takes the fp32 cooperative kernels; the rest the tcgen05 clusters -- Bc = 4 / 10 / 16 /
# 25 rows per batch group, H = 384 (12-CTA clusters: the forward's issue loop ends on a partial group, the backward
# runs the global-ring kernel with 192-column groups), T = 1 (single-step barrier arming)
GRU_CASES = [(50, 64, 64, 6, 4), (1000, 128, 128, 32, 16), (4000, 256, 256, 24, 40), (32768, 512, 512, 128, 64),
             (2000, 128, 384, 16, 50), (100, 128, 128, 1, 8)]


@pytest.mark.parametrize("V,E,H,T,B", GRU_CASES, ids=lambda v: str(v))
def test_gru_loss_and_gradients_match_oracle(session, V, E, H, T, B):
    """Loss, logits and every parameter gradient of one forward/backward at 1e-3 (normwise) against the oracle
    composed from the reference primitives, fed the same bf16 tensor-core operands."""
    from paper_2409_11600_b200 import _lib, autodiff, nn
    from paper_2409_11600_b200.models import GRUClassifier

    rng = np.random.default_rng(V + T)
    tokens = rng.integers(0, V, (B, T)).astype(np.float32)
    y = rng.integers(0, 2, B).astype(np.float32)
    model = GRUClassifier(session, vocab=V, embed=E, hidden=H)
    ref = om.GRUOracle(seed=0, vocab=V, embed=E, hidden=H)
    for (n, t), key in zip(session.param_group.params, ref.order):
        np.testing.assert_array_equal(t.data, ref.params[key])
    tc = bool(_lib.lib().nsk_gru_tc_supported(B, H))
    assert tc == (H >= 128)
    pool = session.pool
    logits = model.forward(autodiff.make_data(pool, tokens))
    dl = logits.data
    loss = nn.cross_entropy(logits, autodiff.make_data(pool, y), pool)
    session.push_named("loss", loss)
    lv = loss.item()
    autodiff.backward(session.tape(), session.grad_cache, pool)
    ref_loss, grads, ref_logits = ref.loss_and_grads(tokens, y, bf16=True, recurrent_bf16=tc)
    assert rel(dl, ref_logits) < 1e-3, rel(dl, ref_logits)
    assert lv == pytest.approx(ref_loss, rel=1e-4)
    for (n, _t), key in zip(session.param_group.params, ref.order):
        e = rel(session.grad_cache.get(n), grads[key])
        assert e < 1e-3, (key, e)


def test_gru_trainer_graph_replay_with_adamw_clip(dev):
    """AdamW + clip_grad_norm step captured as one graph replays like eager (device step counter)."""
    from paper_2409_11600_b200 import nn
    from paper_2409_11600_b200.models import GRUClassifier
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(3)
    V, T, B = 500, 16, 8
    xs = [rng.integers(0, V, (B, T)).astype(np.float32) for _ in range(5)]
    ys = [rng.integers(0, 2, B).astype(np.float32) for _ in range(5)]
    losses = {}
    for mode in (False, True):
        s = Session(seed=0)
        model = GRUClassifier(s, vocab=V, embed=64, hidden=64)
        opt = ("adamw", nn.Hyperparams(learning_rate=1e-3, weight_decay=1e-4), 5.0)
        tr = Trainer(s, model, (B, T), 2, optimizer=opt, graph=mode, warmup=2)
        losses[mode] = [float(tr.step(x, y)) for x, y in zip(xs, ys)]
        if mode:
            assert tr.graph is not None
    np.testing.assert_allclose(losses[True], losses[False], rtol=1e-5)


def test_gru_step_async_matches_step(dev):
    """Token models through Trainer.step_async (two input slots, copy stream, two captured graphs): the second slot's
    token ids are range-checked on the host at staging like the first (no device check inside a capture); losses
    equal Trainer.step's."""
    from paper_2409_11600_b200 import nn
    from paper_2409_11600_b200.models import GRUClassifier
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(21)
    V, B, T = 1000, 16, 12
    xs = [rng.integers(0, V, (B, T)).astype(np.float32) for _ in range(6)]
    ys = [rng.integers(0, 2, B).astype(np.float32) for _ in range(6)]
    out = {}
    for mode in ("step", "async"):
        s = Session(seed=0)
        opt = ("adamw", nn.Hyperparams(learning_rate=1e-3, weight_decay=1e-4), 5.0)
        tr = Trainer(s, GRUClassifier(s, vocab=V, embed=128, hidden=128), (B, T), 2, optimizer=opt, graph=True,
                     warmup=2)
        fn = tr.step if mode == "step" else tr.step_async
        out[mode] = [float(fn(x, y)) for x, y in zip(xs, ys)]
    np.testing.assert_allclose(out["async"], out["step"], rtol=1e-5)
    bad = xs[0].copy()
    bad[3, 4] = V  # out of range: the reference's onehot message, raised at staging
    with pytest.raises(Exception, match="onehot index"):
        tr.step_async(bad, ys[0])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_embedding_gather_equals_reference_onehot_matmul(session, dtype):
    """the embedding gather is the reference's onehot(tokens) @ E (tensor.py:299-317 then the
    float64 matmul_t, tensor.py:213-229) -- a one-term float64 sum, so the float32 gather must match it bit for bit
    (bf16 output: its rounding); the scatter-add backward equals onehot^T . dout to float32 rounding (repeated
    tokens included), time-major rows (row t*B + b holds token [b, t])."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16, F32

    rng = np.random.default_rng(31)
    V, E, B, T = 500, 64, 8, 24
    tokens = rng.integers(0, V, (B, T)).astype(np.float32)
    tokens[0, :5] = 7  # repeated ids: several rows accumulate into one table row
    table = rng.standard_normal((V, E)).astype(np.float32)
    pool = session.pool
    tt = autodiff.make_param(pool, table, "E")
    out = layers.embedding(autodiff.make_data(pool, tokens), tt, pool, dtype=BF16 if dtype == "bf16" else F32)
    onehot = np.zeros((B * T, V))
    tm = tokens.T.reshape(-1).astype(np.int64)  # time-major
    onehot[np.arange(B * T), tm] = 1.0
    ref = onehot @ table.astype(np.float64)  # the reference composition in float64
    want = X.round_bf16(ref) if dtype == "bf16" else ref.astype(np.float32)
    np.testing.assert_array_equal(out.data.reshape(B * T, E), want)
    g = X.round_bf16(rng.standard_normal((B * T, E))) if dtype == "bf16" else rng.standard_normal((B * T, E)).astype(
        np.float32)
    gt = autodiff.make_data(pool, g, dtype=BF16 if dtype == "bf16" else F32)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", out, gt, pool), pool)
    autodiff.push_assignment(session.tape(), "loss", loss)
    autodiff.backward(session.tape(), session.grad_cache, pool)
    dref = onehot.T @ g.astype(np.float64)
    np.testing.assert_allclose(session.grad_cache.get("E"), dref, rtol=1e-6, atol=1e-6)
