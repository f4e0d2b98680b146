"""Cross-check of the restated oracle against torch-CPU float64 autograd (independent second opinion)."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import models as om
from oracle import restated as X


def _t(a):
    return torch.tensor(np.asarray(a, np.float64), requires_grad=True)


def torch_resnet18_loss(params, order, blocks, x_nchw, y):
    P = {k: _t(v) for k, v in params.items()}

    def conv(h, k, st, pad):
        w = P[k].permute(0, 3, 1, 2)  # KRSC -> KCRS
        return F.conv2d(h, w, stride=st, padding=pad)

    def bn(h, k, relu, res=None):
        g, b = P[k][0], P[k][1]
        out = F.batch_norm(h, None, None, g, b, training=True, eps=1e-5)
        if res is not None:
            out = out + res
        return F.relu(out) if relu else out

    x = torch.tensor(x_nchw, dtype=torch.float64)
    h = bn(conv(x, "stem_w", 1, 1), "stem_bn", True)
    for pre, st, proj in blocks:
        o = bn(conv(h, pre + "w1", st, 1), pre + "bn1", True)
        sc = bn(conv(h, pre + "wsc", st, 0), pre + "bnsc", False) if proj else h
        h = bn(conv(o, pre + "w2", 1, 1), pre + "bn2", True, res=sc)
    feat = h.mean(dim=(2, 3))
    logits = feat @ P["fc_w"].T + P["fc_b"]
    loss = F.cross_entropy(logits, torch.tensor(y, dtype=torch.int64))
    loss.backward()
    return float(loss), {k: P[k].grad.numpy() for k in order}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-30))


def test_resnet18_oracle_gradients_match_torch_f64():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((4, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, 4).astype(np.float32)
    ref = om.ResNet18Oracle(seed=0)
    loss, grads, _ = ref.loss_and_grads(x, y, bf16=False)
    tl, tg = torch_resnet18_loss(ref.params, ref.order, ref.blocks, x, y)
    assert loss == pytest.approx(tl, rel=1e-6)
    worst = sorted(((rel(grads[k], tg[k]), k) for k in ref.order), reverse=True)
    assert worst[0][0] < 1e-4, worst[:5]


def test_conv_and_bn_restatements_match_torch():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 9, 9, 8))
    w = rng.standard_normal((5, 3, 3, 8))
    for st, pad in ((1, 1), (2, 1), (2, 0)):
        xt, wt = _t(x), _t(w)
        yt = F.conv2d(xt.permute(0, 3, 1, 2), wt.permute(0, 3, 1, 2), stride=st, padding=pad).permute(0, 2, 3, 1)
        y = X.conv2d_fwd(x, w, st, pad)
        np.testing.assert_allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
        gy = rng.standard_normal(y.shape)
        yt.backward(torch.tensor(gy))
        np.testing.assert_allclose(X.conv2d_dgrad(gy, w, x.shape, st, pad), xt.grad.numpy(), rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(X.conv2d_wgrad(x, gy, w.shape, st, pad), wt.grad.numpy(), rtol=1e-10, atol=1e-10)
    g, b = rng.uniform(0.5, 1.5, 8), rng.uniform(-1, 1, 8)
    r = rng.standard_normal(x.shape)
    xt, gt, bt, rt = _t(x), _t(g), _t(b), _t(r)
    yt = F.relu(F.batch_norm(xt.reshape(-1, 8), None, None, gt, bt, training=True, eps=1e-5).reshape(x.shape) + rt)
    y, cache = X.batchnorm_fwd(x, g, b, relu=True, residual=r)
    np.testing.assert_allclose(y, yt.detach().numpy(), rtol=1e-10, atol=1e-10)
    gy = rng.standard_normal(x.shape)
    yt.backward(torch.tensor(gy))
    dx, dg, db, dres = X.batchnorm_bwd(gy, cache, y_out=y, relu=True)
    np.testing.assert_allclose(dx, xt.grad.numpy(), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(dg, gt.grad.numpy(), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(db, bt.grad.numpy(), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(dres, rt.grad.numpy(), rtol=1e-8, atol=1e-10)


def torch_resnet50_loss(params, order, blocks, x_nchw, y):
    P = {k: _t(v) for k, v in params.items()}

    def conv(h, k, st, pad):
        return F.conv2d(h, P[k].permute(0, 3, 1, 2), stride=st, padding=pad)

    def bn(h, k, relu, res=None):
        out = F.batch_norm(h, None, None, P[k][0], P[k][1], training=True, eps=1e-5)
        if res is not None:
            out = out + res
        return F.relu(out) if relu else out

    x = torch.tensor(x_nchw, dtype=torch.float64)
    h = F.max_pool2d(bn(conv(x, "stem_w", 2, 3), "stem_bn", True), 3, 2, 1)
    for pre, st, proj in blocks:
        o = bn(conv(h, pre + "w1", 1, 0), pre + "bn1", True)
        o = bn(conv(o, pre + "w2", st, 1), pre + "bn2", True)
        sc = bn(conv(h, pre + "wsc", st, 0), pre + "bnsc", False) if proj else h
        h = bn(conv(o, pre + "w3", 1, 0), pre + "bn3", True, res=sc)
    logits = h.mean(dim=(2, 3)) @ P["fc_w"].T + P["fc_b"]
    loss = F.cross_entropy(logits, torch.tensor(y, dtype=torch.int64))
    loss.backward()
    return float(loss), {k: P[k].grad.numpy() for k in order}


def test_resnet50_oracle_matches_torch_f64():
    """C4 oracle (v1.5 bottlenecks, 7x7/2 stem, 3x3/2 max-pool) vs torch autograd at a reduced 64x64 input."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3, 64, 64)).astype(np.float32)
    y = rng.integers(0, 1000, 2).astype(np.float32)
    ref = om.ResNet50Oracle(seed=0)
    assert sum(v.size for v in ref.params.values()) == 25_557_032
    loss, grads, _ = ref.loss_and_grads(x, y, bf16=False)
    tl, tg = torch_resnet50_loss(ref.params, ref.order, ref.blocks, x, y)
    assert loss == pytest.approx(tl, rel=1e-6)
    worst = sorted(((rel(grads[k], tg[k]), k) for k in ref.order), reverse=True)
    assert worst[0][0] < 1e-4, worst[:5]
