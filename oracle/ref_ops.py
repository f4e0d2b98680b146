"""Numpy restatement of the reference's hot-path arithmetic (TEST INFRASTRUCTURE ONLY).

Every function cites the reference line it follows (paths under
/root/reference/pkg/src/nsk/). float32 storage, float64 accumulation, exactly
as the reference: results agree with the reference bit-for-bit except where
BLAS summation order differs (the reference's own tests accept 1e-5 there,
test_tensor.py:142-151). Pinned by tests/test_oracle_golden.py against
vectors produced by the real reference (tests/golden/gen_golden.py).
"""

from __future__ import annotations

import math

import numpy as np


def matmul_t(x, w):
    """y = x . w^T, float64 accumulate, float32 store (tensor.py:213-229)."""
    return (np.asarray(x, np.float32).astype(np.float64) @ np.asarray(w, np.float32).astype(np.float64).T
            ).astype(np.float32)


def plain_matmul(a, b):
    """Untransposed product used by gradient rules (tensor.py:232-234)."""
    return (np.asarray(a, np.float32).astype(np.float64) @ np.asarray(b, np.float32).astype(np.float64)
            ).astype(np.float32)


def stable_sigmoid(z):
    """float64 piecewise-stable sigmoid (tensor.py:237-244)."""
    z = np.asarray(z, np.float32).astype(np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out.astype(np.float32)


def elementwise(kind, a, b=None):
    """tensor.py:247-283 (float32 arithmetic; sigmoid in float64)."""
    a = np.asarray(a, np.float32)
    if kind == "add":
        return a + np.asarray(b, np.float32)
    if kind == "sub":
        return a - np.asarray(b, np.float32)
    if kind == "hadamard":
        return a * np.asarray(b, np.float32)
    if kind == "scalar-add":
        return a + np.float32(b)
    if kind == "scalar-mul":
        return a * np.float32(b)
    if kind == "relu":
        return np.maximum(a, np.float32(0.0))
    if kind == "sigmoid":
        return stable_sigmoid(a)
    if kind == "tanh":
        return np.tanh(a)
    if kind == "neg":
        return -a
    raise ValueError(kind)


def elementwise_grad(kind, g, saved=None, scalar=None):
    """gradient_rule for unary kinds (autodiff.py:268-281)."""
    g = np.asarray(g, np.float32)
    if kind == "relu":
        return (g * (np.asarray(saved) > 0)).astype(np.float32)
    if kind == "sigmoid":
        s = np.asarray(saved, np.float32)
        return (g * s * (1.0 - s)).astype(np.float32)
    if kind == "tanh":
        t = np.asarray(saved, np.float32)
        return (g * (1.0 - t * t)).astype(np.float32)
    if kind == "scalar-mul":
        return (g * np.float32(scalar)).astype(np.float32)
    if kind == "neg":
        return -g
    raise ValueError(kind)


def bias_add(x, b):
    """tensor.py:286-296."""
    return np.asarray(x, np.float32) + np.asarray(b, np.float32)[None, :]


def onehot(idx, classes):
    """tensor.py:299-317 (range errors raise with the row number)."""
    idx = np.asarray(idx, np.float32)
    for row, v in enumerate(idx):
        if v < 0 or v >= classes or v != int(v):
            raise ValueError(f"onehot index {float(v):g} out of range [0, {classes}) at row {row}")
    out = np.zeros((idx.shape[0], classes), np.float32)
    out[np.arange(idx.shape[0]), idx.astype(np.int64)] = 1.0
    return out


def cross_entropy(logits, targets):
    """Returns (loss: float, probs: float32) (autodiff.py:220-248)."""
    z = np.asarray(logits, np.float32).astype(np.float64)
    m = z.shape[0]
    z = z - z.max(axis=1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=1, keepdims=True))
    idx = np.asarray(targets, np.float32).astype(np.int64)
    loss = float(np.mean(lse[:, 0] - z[np.arange(m), idx]))
    return loss, np.exp(z - lse).astype(np.float32)


def cross_entropy_grad(probs, targets, g=1.0):
    """(probs - onehot) * g / m in float64 (autodiff.py:286-292)."""
    m = probs.shape[0]
    d = np.asarray(probs, np.float32).astype(np.float64).copy()
    d[np.arange(m), np.asarray(targets, np.float32).astype(np.int64)] -= 1.0
    d *= float(g) / m
    return d.astype(np.float32)


def sum_loss(x):
    """float64 sum (autodiff.py:213-217)."""
    return float(np.asarray(x, np.float32).astype(np.float64).sum())


def xavier_uniform(rows, cols, seed):
    """nn.py:60-71."""
    a = math.sqrt(6.0 / (rows + cols))
    return np.random.default_rng(seed).uniform(-a, a, size=(rows, cols)).astype(np.float32)


def sgd_update(w, g, v, lr, momentum):
    """v <- mu*v + g ; w <- w - lr*v, float64 math, float32 store (nn.py:91-99). Returns (w, v)."""
    g64 = np.asarray(g, np.float32).reshape(-1).astype(np.float64)
    v64 = momentum * np.asarray(v, np.float32).reshape(-1).astype(np.float64) + g64
    w_new = (np.asarray(w, np.float32).reshape(-1).astype(np.float64) - lr * v64).astype(np.float32)
    return w_new.reshape(np.shape(w)), v64.astype(np.float32).reshape(np.shape(w))


def adamw_update(w, g, m, v, t, lr, wd, b1=0.9, b2=0.999, eps=1e-8):
    """Decoupled decay then bias-corrected Adam, float64 math (nn.py:102-119). Returns (w, m, v)."""
    shape = np.shape(w)
    g64 = np.asarray(g, np.float32).reshape(-1).astype(np.float64)
    w64 = np.asarray(w, np.float32).reshape(-1).astype(np.float64) * (1.0 - lr * wd)
    m64 = b1 * np.asarray(m, np.float32).reshape(-1).astype(np.float64) + (1.0 - b1) * g64
    v64 = b2 * np.asarray(v, np.float32).reshape(-1).astype(np.float64) + (1.0 - b2) * g64 * g64
    mh = m64 / (1.0 - b1 ** t)
    vh = v64 / (1.0 - b2 ** t)
    w_new = (w64 - lr * mh / (np.sqrt(vh) + eps)).astype(np.float32)
    return w_new.reshape(shape), m64.astype(np.float32).reshape(shape), v64.astype(np.float32).reshape(shape)


def clip_grad_norm(grads: list, max_norm: float):
    """Global float64 L2 over all grads; scale in float32 when above max (nn.py:122-139). In place; returns scale."""
    total = 0.0
    for g in grads:
        total += float(np.sum(np.asarray(g).astype(np.float64) ** 2))
    norm = math.sqrt(total)
    if norm <= max_norm:
        return 1.0
    scale = max_norm / norm
    for g in grads:
        g *= np.float32(scale)
    return scale


def accuracy(logits, labels):
    """numpy argmax (first max wins) vs int64 labels, float64 mean (builtins.py:70-80)."""
    pred = np.asarray(logits).argmax(axis=1)
    return float(np.mean(pred == np.asarray(labels, np.float32).astype(np.int64)))


def epoch_permutation(seed: int, num_rows: int, epochs: int, shuffle: bool = True):
    """Per-epoch permutations from one Generator created once (dataset.py:93-102)."""
    rng = np.random.default_rng(seed)
    return [rng.permutation(num_rows) if shuffle else np.arange(num_rows) for _ in range(epochs)]


def batch_rows(perm, index: int, batch_size: int):
    """Contiguous slice of the epoch permutation, partial last batch kept (dataset.py:114-121)."""
    lo = index * batch_size
    return perm[lo:min(lo + batch_size, len(perm))]
