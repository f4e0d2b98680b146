"""Per-op parity: each libnskb kernel (through the drop-in API) vs the CPU oracle on the same inputs.

Tolerances: integer / index work bit-exact; float32 ops with float64 accumulation
at 1e-5 (the reference's own bar, test_tensor.py:142-151); tensor-core ops with
bf16 inputs compare against an oracle fed the same bf16-rounded operands, at a
normwise relative error of 1e-3 after rounding the oracle's output to the
device storage precision (the north star's per-op bar).
"""

import numpy as np
import pytest

from oracle import ref_ops as R
from oracle import restated as X

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture
def pool(dev):
    from paper_2409_11600_b200.tensor import Pool

    return Pool(poison=True)


def dev_tensor(pool, a, bf16=False):
    from paper_2409_11600_b200._lib import BF16, F32
    from paper_2409_11600_b200.tensor import tensor_from_array

    return tensor_from_array(pool, a, dtype=BF16 if bf16 else F32)


# --- GEMM --------------------------------------------------------------------------------------

def naive_matmul_t(x, w):
    m, k = x.shape
    n = w.shape[0]
    out = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            acc = 0.0
            for c in range(k):
                acc += float(x[i, c]) * float(w[j, c])
            out[i, j] = acc
    return out


def test_matmul_t_small_shapes_match_naive_oracle(pool):
    """test_tensor.py:142-151 restated: 100 random shapes, atol 1e-5 (exact fp64-accumulate SIMT path)."""
    from paper_2409_11600_b200.tensor import matmul_t

    rng = np.random.default_rng(42)
    for _ in range(100):
        m, k, n = rng.integers(1, 8, size=3)
        xv = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        wv = rng.uniform(-1, 1, (n, k)).astype(np.float32)
        y = matmul_t(dev_tensor(pool, xv), dev_tensor(pool, wv), pool)
        np.testing.assert_allclose(y.data, naive_matmul_t(xv, wv), atol=1e-5)


def test_matmul_t_known_answers(pool):
    from paper_2409_11600_b200.errors import NskTypeError
    from paper_2409_11600_b200.tensor import matmul_t

    y = matmul_t(dev_tensor(pool, [[1.0, 2.0]]), dev_tensor(pool, [[3.0, 4.0]]), pool)
    assert y.shape == (1, 1) and y.data[0, 0] == pytest.approx(11.0)
    with pytest.raises(NskTypeError) as err:
        matmul_t(dev_tensor(pool, np.zeros((2, 3))), dev_tensor(pool, np.zeros((4, 5))), pool)
    assert "2x3" in str(err.value) and "4x5" in str(err.value)


@pytest.mark.parametrize("m,n,k", [(256, 512, 512), (300, 200, 320), (8192, 1536, 512)])
def test_matmul_t_tf32_tensor_cores(pool, m, n, k):
    """Large f32 products run as tcgen05 kind::tf32; oracle on tf32-rounded (round-to-nearest) inputs."""
    from paper_2409_11600_b200.tensor import matmul_t

    rng = np.random.default_rng(m + n + k)
    xv = rng.standard_normal((m, k)).astype(np.float32)
    wv = rng.standard_normal((n, k)).astype(np.float32)
    y = matmul_t(dev_tensor(pool, xv), dev_tensor(pool, wv), pool).data
    assert rel(y, R.matmul_t(xv, wv)) < 1e-3


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_bf16_all_majorness(dev, a_mn, b_mn):
    """nsk_gemm bf16 operand layouts (K-major / MN-major) through the C ABI."""
    import ctypes as C

    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200._lib import BF16
    from paper_2409_11600_b200.tensor import Buffer

    rng = np.random.default_rng(7)
    M, N, K = 384, 256, 192
    A = X.round_bf16(rng.standard_normal((M, K)))
    B = X.round_bf16(rng.standard_normal((N, K)))
    As = A.T.copy() if a_mn else A
    Bs = B.T.copy() if b_mn else B
    da, db = Buffer(A.size, BF16), Buffer(B.size, BF16)
    da.upload(As)
    db.upload(Bs)
    out = Buffer(M * N)
    out.fill(float("nan"))
    lib = _lib.lib()
    _lib.check(lib.nsk_gemm(BF16, a_mn, b_mn, M, N, K, da.ptr, M if a_mn else K, db.ptr, N if b_mn else K, out.ptr,
                            N, 1, None, 0.0, _lib.stream()))
    got = out.host().reshape(M, N)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    assert rel(got, ref) < 1e-5


# --- conv ----------------------------------------------------------------------------------------

CONV_CASES = [
    (4, 32, 32, 64, 64, 3, 1, 1),
    (4, 32, 32, 64, 128, 3, 2, 1),
    (4, 32, 32, 64, 128, 1, 2, 0),
    (4, 16, 16, 128, 128, 3, 1, 1),
    (8, 8, 8, 256, 256, 3, 1, 1),
    (16, 4, 4, 512, 512, 3, 1, 1),
    (16, 8, 8, 256, 512, 3, 2, 1),
    (3, 32, 32, 3, 64, 3, 1, 1),   # im2col stem (C=3)
    (2, 32, 32, 16, 32, 3, 2, 1),  # im2col small-channel conv with input gradient
]


# ImageNet-shape grids (56/28/14/7 wide): output rows do not tile 128 pixels, so these run through the
# im2col-mode TMA path; odd batches leave a partial last M tile and a K tail in wgrad.
CONV_CASES_I2C = [
    (2, 56, 56, 64, 64, 3, 1, 1),
    (2, 56, 56, 64, 256, 1, 1, 0),
    (2, 56, 56, 128, 128, 3, 2, 1),
    (2, 56, 56, 256, 512, 1, 2, 0),
    (3, 28, 28, 128, 128, 3, 1, 1),
    (4, 14, 14, 256, 256, 3, 1, 1),
    (2, 14, 14, 256, 256, 3, 2, 1),
    (5, 7, 7, 512, 512, 3, 1, 1),
]


@pytest.mark.parametrize("case", CONV_CASES + CONV_CASES_I2C)
def test_conv2d_fprop_dgrad_wgrad(session, case):
    _conv_case(session, case)


@pytest.mark.parametrize("case", CONV_CASES[:7])
def test_conv2d_forced_im2col_mode(session, case, monkeypatch):
    """The im2col-mode TMA path on the CIFAR grids too (NSK_CONV_I2C=1), against the same oracle."""
    monkeypatch.setenv("NSK_CONV_I2C", "1")
    _conv_case(session, case)


def _conv_case(session, case):
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    n, h, w, c, k, r, st, pad = case
    rng = np.random.default_rng(sum(case))
    x = X.round_bf16(rng.standard_normal((n, h, w, c)))
    wt = (rng.standard_normal((k, r, r, c)) / np.sqrt(c * r * r)).astype(np.float32)
    pool = session.pool
    xt = autodiff.make_param(pool, x, "x", dtype=BF16)
    wp = autodiff.make_param(pool, wt, "w")
    y = layers.conv2d(xt, wp, st, pad, pool)
    wq = X.round_bf16(wt)
    ref_y = X.conv2d_fwd(x, wq, st, pad)
    assert rel(y.data, X.round_bf16(ref_y)) < 1e-3
    # backward through the tape: loss = sum(y * gy)
    gy = X.round_bf16(rng.standard_normal(y.shape))
    gyt = autodiff.make_data(pool, gy, dtype=BF16)
    prod = autodiff.rec_elementwise("hadamard", y, gyt, pool)
    loss = autodiff.rec_sum_loss(prod, pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.gy", gyt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)
    # the device gradient of hadamard is g*gy rounded to bf16 (g == 1): exactly gy
    dw_ref = X.conv2d_wgrad(x, gy, wt.shape, st, pad)
    dx_ref = X.conv2d_dgrad(gy, wq, x.shape, st, pad)
    assert rel(session.grad_cache.get("w"), dw_ref) < 1e-3
    assert rel(session.grad_cache.get("x"), X.round_bf16(dx_ref)) < 1e-3


def test_conv2d_shape_errors(session):
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200.errors import NskTypeError

    pool = session.pool
    x = autodiff.make_data(pool, np.zeros((1, 8, 8, 64), np.float32))
    w = autodiff.make_param(pool, np.zeros((64, 3, 3, 32), np.float32), "w")
    with pytest.raises(NskTypeError):
        layers.conv2d(x, w, 1, 1, pool)


# --- batchnorm -------------------------------------------------------------------------------------

@pytest.mark.parametrize("fold_apply", ["0", "1"])
@pytest.mark.parametrize("relu,res", [(False, False), (True, False), (True, True)])
@pytest.mark.parametrize("shape", [(8, 32, 32, 64), (16, 4, 4, 512), (64, 8, 8, 256), (2, 7, 7, 2048)])
def test_batchnorm_fwd_bwd(session, shape, relu, res, fold_apply, monkeypatch):
    """Both finalize strategies: a separate fold kernel, and the fold done by the first blocks of the apply
    pass (NSK_BN_FOLD_APPLY=1; the default for large layers) -- 2048 channels exercise the capped fold grid."""
    monkeypatch.setenv("NSK_BN_FOLD_APPLY", fold_apply)
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    rng = np.random.default_rng(len(shape) + shape[0])
    c = shape[-1]
    pool = session.pool
    x = X.round_bf16(rng.standard_normal(shape) * 2 + 0.5)
    gb = np.stack([rng.uniform(0.5, 1.5, c), rng.uniform(-0.5, 0.5, c)]).astype(np.float32)
    r = X.round_bf16(rng.standard_normal(shape)) if res else None
    xt = autodiff.make_param(pool, x, "x", dtype=BF16)
    gbt = autodiff.make_param(pool, gb, "gb")
    rt = autodiff.make_param(pool, r, "r", dtype=BF16) if res else None
    y = layers.batchnorm(xt, gbt, pool, relu=relu, residual=rt)
    ref_y, cache = X.batchnorm_fwd(x, gb[0], gb[1], relu=relu, residual=r)
    yd = y.data
    assert rel(yd, X.round_bf16(ref_y)) < 1e-3
    gy = X.round_bf16(rng.standard_normal(shape))
    gyt = autodiff.make_data(pool, gy, dtype=BF16)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", y, gyt, pool), pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.gy", gyt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)
    dx, dg, db, dres = X.batchnorm_bwd(gy, cache, y_out=yd, relu=relu)
    assert rel(session.grad_cache.get("gb"), np.stack([dg, db])) < 1e-3
    assert rel(session.grad_cache.get("x"), X.round_bf16(dx)) < 1e-3
    if res:
        assert rel(session.grad_cache.get("r"), X.round_bf16(dres)) < 1e-3


# --- elementwise / bias / onehot -----------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["add", "sub", "hadamard", "scalar-add", "scalar-mul", "relu", "sigmoid", "tanh",
                                  "neg"])
def test_elementwise_fwd_matches_reference(pool, kind):
    from paper_2409_11600_b200.tensor import elementwise

    rng = np.random.default_rng(3)
    a = rng.uniform(-3, 3, (37, 53)).astype(np.float32)
    b = rng.uniform(-3, 3, (37, 53)).astype(np.float32)
    other = dev_tensor(pool, b) if kind in ("add", "sub", "hadamard") else (1.75 if "scalar" in kind else None)
    got = elementwise(kind, dev_tensor(pool, a), other, pool).data
    ref = R.elementwise(kind, a, b if kind in ("add", "sub", "hadamard") else other)
    np.testing.assert_allclose(got, ref, rtol=2e-7, atol=2e-7)


def test_elementwise_known_answers(pool):
    from paper_2409_11600_b200.tensor import elementwise

    np.testing.assert_allclose(
        elementwise("add", dev_tensor(pool, [1.0, 2.0]), dev_tensor(pool, [3.0, 4.0]), pool).data, [4.0, 6.0])
    np.testing.assert_allclose(elementwise("relu", dev_tensor(pool, [-1.0, 0.0, 2.0]), None, pool).data,
                               [0.0, 0.0, 2.0])
    np.testing.assert_allclose(elementwise("sigmoid", dev_tensor(pool, [0.0]), None, pool).data, [0.5])
    ext = elementwise("sigmoid", dev_tensor(pool, [-1000.0, 1000.0]), None, pool).data
    assert np.isfinite(ext).all()
    np.testing.assert_allclose(ext, [0.0, 1.0], atol=1e-6)


def test_bias_add_and_onehot(pool):
    from paper_2409_11600_b200.errors import NskRuntimeError
    from paper_2409_11600_b200.tensor import bias_add, onehot

    np.testing.assert_allclose(
        bias_add(dev_tensor(pool, [[1.0, 2.0], [3.0, 4.0]]), dev_tensor(pool, [10.0, 20.0]), pool).data,
        [[11.0, 22.0], [13.0, 24.0]])
    np.testing.assert_allclose(onehot(dev_tensor(pool, [0.0, 2.0]), 3, pool).data, [[1, 0, 0], [0, 0, 1]])
    with pytest.raises(NskRuntimeError) as err:
        onehot(dev_tensor(pool, [3.0]), 3, pool)
    assert "row 0" in str(err.value)


# --- losses / metrics ----------------------------------------------------------------------------------

@pytest.mark.parametrize("m,c", [(32, 10), (256, 10), (64, 2), (256, 1000), (5, 7)])
def test_cross_entropy_fwd_bwd(session, m, c):
    from paper_2409_11600_b200 import autodiff

    rng = np.random.default_rng(m * c)
    z = rng.uniform(-4, 4, (m, c)).astype(np.float32)
    t = rng.integers(0, c, m).astype(np.float32)
    pool = session.pool
    zt = autodiff.make_param(pool, z, "z")
    tt = autodiff.make_data(pool, t)
    loss = autodiff.rec_cross_entropy(zt, tt, pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t", tt)
    autodiff.push_assignment(tape, "loss", loss)
    ref_loss, probs = R.cross_entropy(z, t)
    lv = loss.item()
    autodiff.backward(tape, session.grad_cache, pool)
    assert lv == pytest.approx(ref_loss, rel=1e-6)
    np.testing.assert_allclose(session.grad_cache.get("z"), R.cross_entropy_grad(probs, t), rtol=1e-5, atol=1e-7)


def test_cross_entropy_known_answers(session):
    from paper_2409_11600_b200 import autodiff
    from paper_2409_11600_b200.errors import NskRuntimeError

    pool = session.pool
    loss = autodiff.rec_cross_entropy(autodiff.make_data(pool, [[0.0, 0.0]]), autodiff.make_data(pool, [1.0]), pool)
    assert loss.item() == pytest.approx(np.log(2.0))
    big = autodiff.rec_cross_entropy(autodiff.make_data(pool, [[1000.0, -1000.0]]),
                                     autodiff.make_data(pool, [0.0]), pool)
    assert np.isfinite(big.item())
    with pytest.raises(NskRuntimeError) as err:
        autodiff.rec_cross_entropy(autodiff.make_data(pool, [[0.0, 0.0]]), autodiff.make_data(pool, [2.0]), pool)
    assert "out of range" in str(err.value) and "row 0" in str(err.value)


def test_accuracy_argmax_bit_exact(session):
    """numpy argmax semantics: first maximum wins, NaN counts as the maximum (builtins.py:70-80)."""
    from paper_2409_11600_b200 import autodiff
    from paper_2409_11600_b200.builtins import BUILTINS

    rng = np.random.default_rng(11)
    z = rng.integers(-3, 3, (512, 10)).astype(np.float32)  # many ties
    z[5, 3] = np.nan
    z[9, 0] = np.nan
    z[9, 7] = np.nan
    y = rng.integers(0, 10, 512).astype(np.float32)
    y[5], y[9] = 3, 0
    pool = session.pool
    got = BUILTINS["accuracy"](session, None, [autodiff.make_data(pool, z), autodiff.make_data(pool, y)], 1)
    assert got == R.accuracy(z, y)


# --- optimizers ------------------------------------------------------------------------------------------

def _group_with_grads(session, shapes, seed):
    from paper_2409_11600_b200 import autodiff

    rng = np.random.default_rng(seed)
    ws, gs = [], []
    for i, shp in enumerate(shapes):
        w = rng.uniform(-1, 1, shp).astype(np.float32)
        g = rng.uniform(-1, 1, shp).astype(np.float32)
        t = autodiff.make_param(session.pool, w, f"p{i}")
        session.param_group.add(f"p{i}", t)
        session.grad_cache.accumulate(f"p{i}", autodiff.make_data(session.pool, g))
        ws.append(w)
        gs.append(g)
    return ws, gs


def test_sgd_matches_reference_bitwise(session):
    from paper_2409_11600_b200 import nn

    shapes = [(3, 5), (7,), (64, 33), (2, 2)]
    ws, gs = _group_with_grads(session, shapes, 1)
    vs = [np.zeros_like(w) for w in ws]
    for step in range(3):
        nn.sgd_step(session.param_group, session.grad_cache, 0.1, 0.9)
        for i in range(len(ws)):
            ws[i], vs[i] = R.sgd_update(ws[i], gs[i], vs[i], 0.1, 0.9)
    for (_n, t), w in zip(session.param_group.params, ws):
        np.testing.assert_array_equal(t.data, w)


def test_sgd_closed_form(session):
    """test_nn.py:203-218: w=1, g=1, lr 0.1, mu 0.9 -> 0.9 then 0.71."""
    from paper_2409_11600_b200 import autodiff, nn

    t = autodiff.make_param(session.pool, [1.0], "w")
    session.param_group.add("w", t)
    session.grad_cache.accumulate("w", autodiff.make_data(session.pool, [1.0]))
    nn.sgd_step(session.param_group, session.grad_cache, 0.1, 0.9)
    assert t.data[0] == pytest.approx(0.9)
    nn.sgd_step(session.param_group, session.grad_cache, 0.1, 0.9)
    assert t.data[0] == pytest.approx(0.71)


def test_adamw_ten_steps_matches_reference(session):
    from paper_2409_11600_b200 import nn

    shapes = [(4, 6), (9,)]
    ws, gs = _group_with_grads(session, shapes, 2)
    ms = [np.zeros_like(w) for w in ws]
    vs = [np.zeros_like(w) for w in ws]
    hp = nn.Hyperparams(learning_rate=1e-2, weight_decay=1e-4)
    for t in range(1, 11):
        nn.adamw_step(session.param_group, session.grad_cache, hp)
        for i in range(len(ws)):
            ws[i], ms[i], vs[i] = R.adamw_update(ws[i], gs[i], ms[i], vs[i], t, 1e-2, 1e-4)
    for (_n, tt), w in zip(session.param_group.params, ws):
        np.testing.assert_allclose(tt.data, w, rtol=1e-6, atol=1e-7)


def test_clip_grad_norm(session):
    """test_nn.py:315-340: [6, 8] with max 5 -> [3, 4], scale 0.5; no clip below the max."""
    from paper_2409_11600_b200 import autodiff, nn

    session.grad_cache.accumulate("a", autodiff.make_data(session.pool, [6.0, 8.0]))
    scale = nn.clip_grad_norm(session.grad_cache, 5.0)
    assert float(scale) == pytest.approx(0.5)
    np.testing.assert_allclose(session.grad_cache.get("a"), [3.0, 4.0], rtol=1e-6)
    assert float(nn.clip_grad_norm(session.grad_cache, 10.0)) == 1.0


# --- pooling / layout / augmentation / embedding ----------------------------------------------------------

@pytest.mark.parametrize("relu_ties", [False, True])
def test_avgpool_and_maxpool(session, relu_ties):
    """relu_ties: post-ReLU input (many equal zeros) exercises the first-maximum tie rule, bit for bit."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    rng = np.random.default_rng(5)
    pool = session.pool
    x = X.round_bf16(rng.standard_normal((4, 8, 8, 64)))
    if relu_ties:
        x = np.maximum(x, 0)
    xt = autodiff.make_param(pool, x, "x", dtype=BF16)
    y = layers.avgpool_global(autodiff.make_data(pool, x, dtype=BF16), pool)
    assert rel(y.data, X.avgpool_fwd(x)) < 1e-6
    m = layers.maxpool(xt, 3, 2, 1, pool)
    np.testing.assert_array_equal(m.data, X.maxpool_fwd(x, 3, 2, 1).astype(np.float32))
    gy = X.round_bf16(rng.standard_normal(m.shape))
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", m, autodiff.make_data(pool, gy, dtype=BF16),
                                                          pool), pool)
    autodiff.push_assignment(session.tape(), "loss", loss)
    autodiff.backward(session.tape(), session.grad_cache, pool)
    assert rel(session.grad_cache.get("x"), X.round_bf16(X.maxpool_bwd(x, gy, 3, 2, 1))) < 1e-3


def test_augment_crop_flip_indices_bit_exact(dev):
    import ctypes as C

    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200._lib import BF16, F32
    from paper_2409_11600_b200.tensor import Buffer

    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (16, 32, 32, 3), dtype=np.uint8)
    offs = X.draw_crop_flip(np.random.default_rng(123), 16, pad=4)
    mean = np.array([0.4914, 0.4822, 0.4465], np.float32)
    std = np.array([0.2470, 0.2435, 0.2616], np.float32)
    lib = _lib.lib()
    d_img = Buffer(img.size // 4 + 1, F32)
    _lib.check(lib.nsk_memcpy_h2d(d_img.ptr, img.ctypes.data, img.nbytes, _lib.stream()))
    d_off = Buffer(offs.size, F32)
    _lib.check(lib.nsk_memcpy_h2d(d_off.ptr, offs.ctypes.data, offs.nbytes, _lib.stream()))
    d_ms = Buffer(6, F32)
    d_ms.upload(np.concatenate([mean, std]))
    out = Buffer(16 * 32 * 32 * 8, BF16)
    _lib.check(lib.nsk_augment_crop_flip(d_img.ptr, d_off.ptr, out.ptr, 16, 32, 32, 3, 4, d_ms.ptr, d_ms.ptr + 12, 8,
                                         _lib.stream()))
    got = out.host().reshape(16, 32, 32, 8)
    ref = X.augment_crop_flip(img, offs, 4, mean, std, channels_pad=8)
    # pixel values: the oracle's float64 (u8/255 - mean)/std rounded to bf16 -- at most one bf16 ulp apart (the
    # device divides in fp32), normwise within 1e-3
    refq = X.round_bf16(ref)
    assert rel(got, refq) < 1e-3
    np.testing.assert_allclose(got, refq, rtol=2 ** -7, atol=0)
    # index exactness: zero-padded border pixels land exactly where the oracle puts them
    np.testing.assert_array_equal(got[..., :3] == X.round_bf16(-mean / std), X.round_bf16(ref)[..., :3] ==
                                  X.round_bf16(-mean / std))


@pytest.mark.parametrize("case", [
    (8, 32, 32, 64, 64, 3, 1, 1),      # N=64 row-reuse tiles, 2 CTAs/SM
    (16, 8, 8, 256, 512, 3, 2, 1),     # wide tiles, several n-tiles per CTA
    (2, 28, 28, 128, 128, 3, 1, 1),    # im2col-mode A, partial last M tile
    (4, 7, 7, 512, 2048, 1, 1, 0),     # ResNet-50 expand: 2048 channels of partials
])
def test_conv_bn_fused_statistics(session, case):
    """conv_bn: BN statistics from the conv epilogue's channel partials vs the oracle BN of the stored conv output."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    n, h, w, c, k, r, st, pad = case
    rng = np.random.default_rng(sum(case))
    x = X.round_bf16(rng.standard_normal((n, h, w, c)))
    wt = (rng.standard_normal((k, r, r, c)) / np.sqrt(c * r * r)).astype(np.float32)
    gb = np.stack([rng.uniform(0.5, 1.5, k), rng.uniform(-0.5, 0.5, k)]).astype(np.float32)
    pool = session.pool
    xt = autodiff.make_data(pool, x, dtype=BF16)
    wp = autodiff.make_param(pool, wt, "w")
    gbt = autodiff.make_param(pool, gb, "gb")
    conv = layers.conv2d(xt, wp, st, pad, pool, bn_stats=True)
    assert conv.bn_partials is not None
    cdata = conv.data.astype(np.float64)
    y = layers.batchnorm(conv, gbt, pool, relu=True)
    ref, (_xhat, invstd, _g, mean) = X.batchnorm_fwd(cdata, gb[0], gb[1], relu=True)
    assert rel(y.data, X.round_bf16(ref)) < 1e-3
    assert conv.bn_partials is None  # consumed and returned to the pool
    node_saved = y.node.saved
    np.testing.assert_allclose(node_saved[2].data, mean, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(node_saved[3].data, invstd, rtol=1e-4)


@pytest.mark.parametrize("case", [(4, 32, 32, 64, 64, 3, 1, 1), (2, 56, 56, 256, 64, 1, 1, 0),
                                  (4, 32, 32, 64, 128, 3, 2, 1), (4, 32, 32, 64, 128, 1, 2, 0),
                                  (2, 14, 14, 128, 256, 1, 2, 0)])
def test_conv2d_dgrad_accumulates_in_place(dev, case):
    """nsk_conv2d_dgrad_acc: dx = dgrad + dx (TMA reduce-add for stride 1, staged read-modify-write for the
    stride-2 parity classes) -- the in-place second gradient contribution the autodiff uses. 1x1 stride 2:
    only parity class (0, 0) has a tap; the other three are dropped and must leave dx untouched."""
    import ctypes as C

    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200._lib import BF16, ConvDesc
    from paper_2409_11600_b200.tensor import Buffer

    n, h, w, c, k, r, st, pad = case
    p = (h + 2 * pad - r) // st + 1
    rng = np.random.default_rng(sum(case))
    dy = X.round_bf16(rng.standard_normal((n, p, p, k)))
    wt = X.round_bf16(rng.standard_normal((k, r, r, c)) / np.sqrt(k * r * r))
    dx0 = X.round_bf16(rng.standard_normal((n, h, w, c)))
    bufs = {}
    for name, a in (("dy", dy), ("w", wt), ("dx", dx0)):
        bufs[name] = Buffer(a.size, BF16)
        bufs[name].upload(a)
    d = ConvDesc(n, h, w, c, k, r, r, st, pad, p, p)
    lib = _lib.lib()
    _lib.check(lib.nsk_conv2d_dgrad_acc(C.byref(d), bufs["dy"].ptr, bufs["w"].ptr, bufs["dx"].ptr, 1.0,
                                        _lib.stream()))
    got = bufs["dx"].host().reshape(dx0.shape)
    ref = dx0.astype(np.float64) + X.round_bf16(X.conv2d_dgrad(dy, wt, dx0.shape, st, pad))
    assert rel(got, X.round_bf16(ref)) < 1e-3


@pytest.mark.parametrize("case", [(16, 4, 4, 512, 512, 3, 1, 1), (64, 4, 4, 512, 512, 3, 1, 1)])
def test_conv_split_k_matches_unsplit(dev, case, monkeypatch):
    """Split-K conv passes (few output tiles, long reduction: 256-wide tiles + fixed-order fold that also
    writes the BN statistics partials) against the unsplit kernels: outputs and folded statistics agree to
    bf16 rounding (the two sum the same products in different orders)."""
    import ctypes as C

    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200._lib import BF16, F32, ConvDesc
    from paper_2409_11600_b200.tensor import Buffer

    n, h, w, c, k, r, st, pad = case
    p = (h + 2 * pad - r) // st + 1
    rng = np.random.default_rng(sum(case))
    x = X.round_bf16(rng.standard_normal((n, h, w, c)))
    wt = X.round_bf16(rng.standard_normal((k, r, r, c)) / np.sqrt(r * r * c))
    lib = _lib.lib()
    d = ConvDesc(n, h, w, c, k, r, r, st, pad, p, p)
    xb, wb, yb, dxb = Buffer(x.size, BF16), Buffer(wt.size, BF16), Buffer(n * p * p * k, BF16), Buffer(x.size, BF16)
    xb.upload(x)
    wb.upload(wt)
    nst = int(lib.nsk_conv2d_stats_floats(k)) if hasattr(lib, "nsk_conv2d_stats_floats") else 4 * 148 * 2 * k + 8 * k
    parts = Buffer(nst, F32)
    out = {}
    for split in ("1", "0"):
        monkeypatch.setenv("NSK_CONV_SPLIT", split)
        npart = C.c_int(0)
        _lib.check(lib.nsk_conv2d_fprop_stats(C.byref(d), xb.ptr, wb.ptr, yb.ptr, parts.ptr, nst, C.byref(npart),
                                               _lib.stream()))
        y = yb.host().reshape(n, p, p, k).astype(np.float64)
        stats = parts.host()[: npart.value * 2 * k].reshape(npart.value, 2, k).astype(np.float64).sum(0)
        _lib.check(lib.nsk_conv2d_dgrad(C.byref(d), yb.ptr, wb.ptr, dxb.ptr, _lib.stream()))
        out[split] = (y, stats, dxb.host().astype(np.float64).reshape(x.shape))
    ys, ss, ds = out["1"]
    yu, su, du = out["0"]
    assert rel(ys, yu) < 1e-3 and rel(ss, su) < 1e-3
    assert rel(ds, X.round_bf16(X.conv2d_dgrad(yu.astype(np.float32), wt, x.shape, st, pad))) < 1e-3
    assert rel(ds, du) < 1e-3


@pytest.mark.parametrize("case", [(2, 3, 40, 40, 7, 2, 3), (3, 3, 32, 32, 3, 1, 1), (2, 3, 17, 23, 5, 2, 2)])
def test_im2col_nchw_matches_oracle(dev, case):
    """The image stem's fused layout change + im2col (NCHW float32 -> [N*P*Q, Kp] bf16, K = R*S*C zero-padded to a
    multiple of 8), row-tiled through shared memory: bit-exact against the oracle's im2col of the NHWC image, the
    padding columns zero."""
    import ctypes as C

    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200._lib import BF16, F32
    from paper_2409_11600_b200.tensor import Buffer

    n, c, h, w, r, st, pad = case
    p, q = (h + 2 * pad - r) // st + 1, (w + 2 * pad - r) // st + 1
    kp = (r * r * c + 7) // 8 * 8
    rng = np.random.default_rng(sum(case))
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    xb, ob = Buffer(x.size, F32), Buffer(n * p * q * kp, BF16)
    xb.upload(x)
    lib = _lib.lib()
    _lib.check(lib.nsk_im2col_nchw(xb.ptr, ob.ptr, n, c, h, w, r, r, st, pad, p, q, kp, _lib.stream()))
    got = ob.host().reshape(n * p * q, kp)
    ref = X.round_bf16(X.im2col(x.transpose(0, 2, 3, 1), r, r, st, pad)).astype(np.float32)
    np.testing.assert_array_equal(got[:, : r * r * c], ref)
    assert not np.any(got[:, r * r * c:])


@pytest.mark.parametrize("k,st,pad", [(3, 2, 1), (2, 2, 0), (3, 1, 1)])
def test_maxpool_window_variants(session, k, st, pad):
    """Max-pool forward (bit-exact, first-maximum ties) and backward for the compile-time 3x3/2 kernels and the
    runtime-window fallback."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    rng = np.random.default_rng(k * 10 + st)
    pool = session.pool
    x = np.maximum(X.round_bf16(rng.standard_normal((3, 9, 11, 16))), 0)  # ReLU'd: many ties
    xt = autodiff.make_param(pool, x, "x", dtype=BF16)
    m = layers.maxpool(xt, k, st, pad, pool)
    np.testing.assert_array_equal(m.data, X.maxpool_fwd(x, k, st, pad).astype(np.float32))
    gy = X.round_bf16(rng.standard_normal(m.shape))
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", m, autodiff.make_data(pool, gy, dtype=BF16),
                                                          pool), pool)
    autodiff.push_assignment(session.tape(), "loss", loss)
    autodiff.backward(session.tape(), session.grad_cache, pool)
    assert rel(session.grad_cache.get("x"), X.round_bf16(X.maxpool_bwd(x, gy, k, st, pad))) < 1e-3
