"""float64 restatements of the hot-path ops the reference lacks (TEST INFRASTRUCTURE ONLY).

The reference has no conv, batchnorm, pooling, augmentation or fused GRU
(pkg/README.md:167-172). These restatements
follow its numeric conventions -- float32 storage, float64 accumulation
(tensor.py:227), losses averaged inside their own rules (autodiff.py:286-292)
-- and are pinned by the reference's finite-difference method
(gradcheck.py:89-138: eps 1e-3, rel 1e-2, abs 1e-4) in tests/test_oracle_fd.py,
plus a torch-CPU float64 cross-check. Parity of these ops against the
reference itself is therefore "pinned by FD" (the reference cannot run them).

Layouts: activations NHWC, filters KRSC (k = output channel), the same as the
device kernels.
"""

from __future__ import annotations

import math

import numpy as np


def round_bf16(a):
    """Round to the nearest bfloat16 (ties to even), returned as float32 -- the device storage format."""
    a32 = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = a32.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16
    out = r.astype(np.uint32).view(np.float32).reshape(a32.shape)
    return np.where(np.isnan(a32), np.float32(np.nan), out)


def conv_out(h, k, stride, pad):
    return (h + 2 * pad - k) // stride + 1


def im2col(x, R, S, stride, pad):
    """[N,H,W,C] -> [N*P*Q, R*S*C] with column index (r*S + s)*C + c (zero padding)."""
    N, H, W, C = x.shape
    P, Q = conv_out(H, R, stride, pad), conv_out(W, S, stride, pad)
    xp = np.pad(np.asarray(x, np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    cols = np.empty((N, P, Q, R, S, C), np.float64)
    for r in range(R):
        for s in range(S):
            cols[:, :, :, r, s, :] = xp[:, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride, :]
    return cols.reshape(N * P * Q, R * S * C)


def col2im(dcols, x_shape, R, S, stride, pad):
    """Adjoint of im2col: scatter-add [N*P*Q, R*S*C] back into [N,H,W,C]."""
    N, H, W, C = x_shape
    P, Q = conv_out(H, R, stride, pad), conv_out(W, S, stride, pad)
    d = np.asarray(dcols, np.float64).reshape(N, P, Q, R, S, C)
    dxp = np.zeros((N, H + 2 * pad, W + 2 * pad, C), np.float64)
    for r in range(R):
        for s in range(S):
            dxp[:, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride, :] += d[:, :, :, r, s, :]
    return dxp[:, pad:pad + H, pad:pad + W, :]


_CHUNK_ELEMS = 1 << 25  # im2col elements per chunk (256 MiB of float64): bench-size batches go image-block-wise


def _image_chunks(n, per_image):
    step = max(1, _CHUNK_ELEMS // max(1, per_image))
    return [(i, min(n, i + step)) for i in range(0, n, step)]


def conv2d_fwd(x, w, stride, pad):
    """y[n,p,q,k] = sum_{r,s,c} x[n, p*st-pad+r, q*st-pad+s, c] * w[k,r,s,c]  (float64)."""
    N, H, W_, _ = x.shape
    K, R, S, C = w.shape
    P, Q = conv_out(H, R, stride, pad), conv_out(W_, S, stride, pad)
    wm = np.asarray(w, np.float64).reshape(K, -1).T
    y = np.empty((N, P, Q, K), np.float64)
    for a, b in _image_chunks(N, P * Q * R * S * C):
        y[a:b] = (im2col(x[a:b], R, S, stride, pad) @ wm).reshape(b - a, P, Q, K)
    return y


def conv2d_dgrad(dy, w, x_shape, stride, pad):
    K, R, S, C = w.shape
    N = x_shape[0]
    wm = np.asarray(w, np.float64).reshape(K, -1)
    P, Q = np.shape(dy)[1], np.shape(dy)[2]
    dx = np.empty(x_shape, np.float64)
    for a, b in _image_chunks(N, P * Q * R * S * C):
        dcols = np.asarray(dy[a:b], np.float64).reshape(-1, K) @ wm
        dx[a:b] = col2im(dcols, (b - a,) + tuple(x_shape[1:]), R, S, stride, pad)
    return dx


def conv2d_wgrad(x, dy, w_shape, stride, pad):
    K, R, S, C = w_shape
    N = x.shape[0]
    P, Q = np.shape(dy)[1], np.shape(dy)[2]
    dw = np.zeros((K, R * S * C), np.float64)
    for a, b in _image_chunks(N, P * Q * R * S * C):
        dw += np.asarray(dy[a:b], np.float64).reshape(-1, K).T @ im2col(x[a:b], R, S, stride, pad)
    return dw.reshape(K, R, S, C)


def batchnorm_fwd(x, gamma, beta, eps=1e-5, relu=False, residual=None):
    """Training-mode BN over all rows (N*H*W) per channel, biased variance; float64.

    Returns (y, cache); cache = (xhat, invstd, gamma, y_out_for_mask)."""
    x2 = np.asarray(x, np.float64).reshape(-1, x.shape[-1])
    mean = x2.mean(axis=0)
    var = ((x2 - mean) ** 2).mean(axis=0)
    invstd = 1.0 / np.sqrt(var + eps)
    xhat = (x2 - mean) * invstd
    y = xhat * np.asarray(gamma, np.float64) + np.asarray(beta, np.float64)
    if residual is not None:
        y = y + np.asarray(residual, np.float64).reshape(y.shape)
    if relu:
        y = np.maximum(y, 0.0)
    return y.reshape(x.shape), (xhat, invstd, np.asarray(gamma, np.float64), mean)


def batchnorm_bwd(dy, cache, y_out=None, relu=False):
    """Returns (dx, dgamma, dbeta, dresidual). dz = dy * [y > 0] when relu."""
    xhat, invstd, gamma, _mean = cache
    shape = np.shape(dy)
    dz = np.asarray(dy, np.float64).reshape(xhat.shape)
    if relu:
        dz = dz * (np.asarray(y_out).reshape(xhat.shape) > 0)
    M = xhat.shape[0]
    dbeta = dz.sum(axis=0)
    dgamma = (dz * xhat).sum(axis=0)
    dx = gamma * invstd * (dz - dbeta / M - xhat * dgamma / M)
    return dx.reshape(shape), dgamma, dbeta, dz.reshape(shape)


def avgpool_fwd(x):
    """[N,H,W,C] -> [N,C] mean over H*W (float64)."""
    return np.asarray(x, np.float64).mean(axis=(1, 2))


def avgpool_bwd(dy, x_shape):
    N, H, W, C = x_shape
    return np.broadcast_to(np.asarray(dy, np.float64)[:, None, None, :] / (H * W), x_shape).copy()


def maxpool_fwd(x, k, stride, pad):
    N, H, W, C = x.shape
    P, Q = conv_out(H, k, stride, pad), conv_out(W, k, stride, pad)
    xp = np.pad(np.asarray(x, np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)), constant_values=-np.inf)
    out = np.full((N, P, Q, C), -np.inf)
    for r in range(k):
        for s in range(k):
            out = np.maximum(out, xp[:, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride, :])
    return out


def maxpool_bwd(x, dy, k, stride, pad):
    """Gradient to the first maximum of each window (row-major window order)."""
    N, H, W, C = x.shape
    P, Q = dy.shape[1], dy.shape[2]
    xp = np.pad(np.asarray(x, np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)), constant_values=-np.inf)
    dxp = np.zeros_like(xp)
    best = np.full((N, P, Q, C), -np.inf)
    arg = np.zeros((N, P, Q, C), np.int64)
    for r in range(k):
        for s in range(k):
            v = xp[:, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride, :]
            upd = v > best
            best = np.where(upd, v, best)
            arg = np.where(upd, r * k + s, arg)
    for r in range(k):
        for s in range(k):
            sel = (arg == r * k + s)
            dxp[:, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride, :] += np.where(sel, dy, 0.0)
    return dxp[:, pad:pad + H, pad:pad + W, :]


def draw_crop_flip(rng: np.random.Generator, n: int, pad: int = 4):
    """Host index draw order shared by device and oracle: per image (dy, dx, flip)."""
    out = np.empty((n, 3), np.int32)
    for i in range(n):
        out[i, 0] = rng.integers(0, 2 * pad + 1)
        out[i, 1] = rng.integers(0, 2 * pad + 1)
        out[i, 2] = rng.integers(0, 2)
    return out


def augment_crop_flip(img_u8, offs, pad, mean, std, channels_pad=None):
    """uint8 NHWC -> zero-padded crop at (dy, dx), optional h-flip, (v/255 - mean)/std; float64."""
    N, H, W, C = img_u8.shape
    cp = channels_pad or C
    out = np.zeros((N, H, W, cp), np.float64)
    raw = np.pad(img_u8.astype(np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    for i in range(N):
        oy, ox, fl = (int(v) for v in offs[i])
        crop = raw[i, oy:oy + H, ox:ox + W, :]
        if fl:
            crop = crop[:, ::-1, :]
        out[i, :, :, :C] = (crop / 255.0 - np.asarray(mean, np.float64)) / np.asarray(std, np.float64)
    return out


def xavier_conv(cout, r, s, cin, seed):
    """KRSC filters, a = sqrt(6 / (cin*r*s + cout*r*s)), default_rng(seed).uniform (nn.py:60-71 restated)."""
    a = math.sqrt(6.0 / (cin * r * s + cout * r * s))
    return np.random.default_rng(seed).uniform(-a, a, size=(cout, r, s, cin)).astype(np.float32)


def embedding_fwd(table, tokens):
    """onehot(tokens) @ E in float64 == E[tokens] exactly (tensor.py:299-317 then :213-229)."""
    return np.asarray(table, np.float32)[np.asarray(tokens, np.int64)]


def embedding_bwd(dout, tokens, vocab):
    d = np.zeros((vocab, dout.shape[-1]), np.float64)
    np.add.at(d, np.asarray(tokens, np.int64).reshape(-1), np.asarray(dout, np.float64).reshape(-1, dout.shape[-1]))
    return d
