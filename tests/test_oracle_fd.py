"""Pin the restated ops (oracle/restated.py) with the reference's own finite-difference method.

gradcheck.py:17-19 and :89-138: central differences, eps 1e-3 in float64, pass when
|analytic - fd| <= 1e-4 + 1e-2 * |fd| for every element. CPU only.
"""

import numpy as np
import pytest

from oracle import restated as X

EPS, REL, ABS = 1e-3, 1e-2, 1e-4


def fd_check(f, args, grads, wrt):
    """f(*args) -> scalar; grads[i] analytic gradient for args[wrt[i]]."""
    for gi, ai in zip(grads, wrt):
        base = args[ai]
        flat = base.reshape(-1)
        fd = np.zeros_like(flat)
        for j in range(flat.size):
            o = flat[j]
            flat[j] = o + EPS
            hi = f(*args)
            flat[j] = o - EPS
            lo = f(*args)
            flat[j] = o
            fd[j] = (hi - lo) / (2 * EPS)
        err = np.abs(np.asarray(gi).reshape(-1) - fd)
        assert (err <= ABS + REL * np.abs(fd)).all(), float((err - ABS - REL * np.abs(fd)).max())


@pytest.mark.parametrize("st,pad,k", [(1, 1, 3), (2, 1, 3), (2, 0, 1), (1, 0, 1)])
def test_conv2d_fd(st, pad, k):
    rng = np.random.default_rng(st * 10 + pad + k)
    x = rng.uniform(-1, 1, (2, 5, 6, 3))
    w = rng.uniform(-1, 1, (4, k, k, 3))
    gy = rng.uniform(-1, 1, X.conv2d_fwd(x, w, st, pad).shape)
    f = lambda x_, w_: float((X.conv2d_fwd(x_, w_, st, pad) * gy).sum())  # noqa: E731
    fd_check(f, [x, w], [X.conv2d_dgrad(gy, w, x.shape, st, pad), X.conv2d_wgrad(x, gy, w.shape, st, pad)], [0, 1])


@pytest.mark.parametrize("relu,res", [(False, False), (True, False), (True, True)])
def test_batchnorm_fd(relu, res):
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (3, 2, 2, 4)) * 2 + 0.3
    g = rng.uniform(0.5, 1.5, 4)
    b = rng.uniform(-0.5, 0.5, 4)
    r = rng.uniform(-1, 1, x.shape)
    gy = rng.uniform(-1, 1, x.shape)

    def f(x_, g_, b_, r_):
        y, _ = X.batchnorm_fwd(x_, g_, b_, relu=relu, residual=r_ if res else None)
        return float((y * gy).sum())

    y, cache = X.batchnorm_fwd(x, g, b, relu=relu, residual=r if res else None)
    dx, dg, db, dres = X.batchnorm_bwd(gy, cache, y_out=y, relu=relu)
    grads, wrt = [dx, dg, db], [0, 1, 2]
    if res:
        grads.append(dres)
        wrt.append(3)
    fd_check(f, [x, g, b, r], grads, wrt)


def test_pooling_fd():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 4, 4, 3))
    gy = rng.uniform(-1, 1, (2, 3))
    fd_check(lambda x_: float((X.avgpool_fwd(x_) * gy).sum()), [x], [X.avgpool_bwd(gy, x.shape)], [0])
    y = X.maxpool_fwd(x, 3, 2, 1)
    gm = rng.uniform(-1, 1, y.shape)
    fd_check(lambda x_: float((X.maxpool_fwd(x_, 3, 2, 1) * gm).sum()), [x], [X.maxpool_bwd(x, gm, 3, 2, 1)], [0])


def test_im2col_col2im_adjoint():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 7, 6, 3))
    cols = X.im2col(x, 3, 3, 2, 1)
    d = rng.standard_normal(cols.shape)
    assert np.isclose((cols * d).sum(), (x * X.col2im(d, x.shape, 3, 3, 2, 1)).sum())


def test_crop_flip_index_draw_is_deterministic():
    a = X.draw_crop_flip(np.random.default_rng(9), 32)
    b = X.draw_crop_flip(np.random.default_rng(9), 32)
    np.testing.assert_array_equal(a, b)
    assert a[:, :2].min() >= 0 and a[:, :2].max() <= 8 and set(np.unique(a[:, 2])) <= {0, 1}
    img = np.arange(2 * 4 * 4 * 1, dtype=np.uint8).reshape(2, 4, 4, 1)
    offs = np.array([[1, 1, 0], [1, 1, 1]], np.int32)  # centred crop (pad 1), second image flipped
    out = X.augment_crop_flip(img, offs, 1, [0.0], [1.0 / 255.0])
    np.testing.assert_array_equal(out[0, :, :, 0], img[0, :, :, 0])
    np.testing.assert_array_equal(out[1, :, :, 0], img[1, :, ::-1, 0])


def test_round_bf16_ties_to_even():
    vals = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, -2.5, 0.0, np.inf], np.float32)
    got = X.round_bf16(vals)
    np.testing.assert_array_equal(got, np.array([1.0, 1.0, 1.0 + 2**-6, -2.5, 0.0, np.inf], np.float32))
