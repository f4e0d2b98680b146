"""Per-op parity at the BASELINE configuration C2 (ResNet-18/CIFAR, batch 256): every distinct conv geometry of
the network at N = 256, through the same layer calls the training step makes, against the float64 oracle fed
the same bf16 operands.

At N = 256 each persistent CTA walks many tiles: the weight-resident fprop, the row-reuse (rr64 / rr128)
weight-gradient kernels, the TMEM double-buffered tile loop and the split-K folds all run exactly as in the
bench, which the small-N cases in test_gpu_ops.py do not reach.

Bar: the north star's 1e-3 normwise relative error per op (bf16 inputs, fp32 accumulation), the oracle's
output rounded to the device's storage precision (bf16 activations, fp32 weight gradients).
"""

import numpy as np
import pytest

from oracle import restated as X

pytestmark = pytest.mark.gpu

B = 256
TOL = 1e-3

# (H=W, Cin, Cout, R, stride, pad) of every distinct conv in ResNet-18/CIFAR
C2_CONVS = [
    (32, 64, 64, 3, 1, 1),     # layer1 3x3 (x4)
    (32, 64, 128, 3, 2, 1),    # layer2 first conv1
    (32, 64, 128, 1, 2, 0),    # layer2 projection shortcut
    (16, 128, 128, 3, 1, 1),   # layer2 3x3 (x3)
    (16, 128, 256, 3, 2, 1),   # layer3 first conv1
    (16, 128, 256, 1, 2, 0),   # layer3 projection shortcut
    (8, 256, 256, 3, 1, 1),    # layer3 3x3 (x3)
    (8, 256, 512, 3, 2, 1),    # layer4 first conv1
    (8, 256, 512, 1, 2, 0),    # layer4 projection shortcut
    (4, 512, 512, 3, 1, 1),    # layer4 3x3 (x3)
]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _ids(c):
    hw, ci, co, r, st, _p = c
    return f"{hw}x{hw}_{ci}to{co}_{r}x{r}_s{st}"


@pytest.mark.parametrize("case", C2_CONVS, ids=_ids)
def test_conv_bn_chain_at_batch_256(session, case):
    """conv2d (BN statistics fused into the tcgen05 epilogue) -> batchnorm(+ReLU) forward, then the backward
    chain BN -> dgrad / wgrad (wgrad forked onto the side stream), at the bench batch."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    hw, c, k, r, st, pad = case
    rng = np.random.default_rng(1000 + sum(case))
    x = X.round_bf16(rng.standard_normal((B, hw, hw, c)))
    wt = (rng.standard_normal((k, r, r, c)) * np.sqrt(2.0 / (c * r * r))).astype(np.float32)
    gb = np.stack([rng.uniform(0.5, 1.5, k), rng.uniform(-0.5, 0.5, k)]).astype(np.float32)
    pool = session.pool
    xt = autodiff.make_param(pool, x, "x", dtype=BF16)
    wp = autodiff.make_param(pool, wt, "w")
    gbt = autodiff.make_param(pool, gb, "gb")
    conv = layers.conv2d(xt, wp, st, pad, pool, bn_stats=True)
    y = layers.batchnorm(conv, gbt, pool, relu=True)
    conv_d, y_d = conv.data, y.data

    wq = X.round_bf16(wt)
    ref_c = X.round_bf16(X.conv2d_fwd(x, wq, st, pad))
    assert rel(conv_d, ref_c) < TOL, ("conv y", rel(conv_d, ref_c))
    ref_y, cache = X.batchnorm_fwd(ref_c, gb[0], gb[1], relu=True)
    assert rel(y_d, X.round_bf16(ref_y)) < TOL, ("bn y", rel(y_d, X.round_bf16(ref_y)))

    gy = X.round_bf16(rng.standard_normal(y.shape))
    gyt = autodiff.make_data(pool, gy, dtype=BF16)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", y, gyt, pool), pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.gy", gyt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)

    dc, dg, db, _ = X.batchnorm_bwd(gy, cache, y_out=y_d, relu=True)
    dcq = X.round_bf16(dc)  # the device stores the conv-output gradient as bf16
    got_gb = session.grad_cache.get("gb")
    assert rel(got_gb, np.stack([dg, db])) < TOL, ("dgamma/dbeta", rel(got_gb, np.stack([dg, db])))
    dw_ref = X.conv2d_wgrad(x, dcq, wt.shape, st, pad)
    got_dw = session.grad_cache.get("w")
    assert rel(got_dw, dw_ref) < TOL, ("dw", rel(got_dw, dw_ref))
    dx_ref = X.round_bf16(X.conv2d_dgrad(dcq, wq, x.shape, st, pad))
    got_dx = session.grad_cache.get("x")
    assert rel(got_dx, dx_ref) < TOL, ("dx", rel(got_dx, dx_ref))


@pytest.mark.parametrize("case", C2_CONVS, ids=_ids)
def test_conv_passes_at_batch_256(session, case, monkeypatch, pair_multicast=False):
    """The three conv passes alone (no BN between): fprop, dgrad, wgrad with a random bf16 output gradient."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    if pair_multicast:
        monkeypatch.setenv("NSK_MC", "1")

    hw, c, k, r, st, pad = case
    rng = np.random.default_rng(2000 + sum(case))
    x = X.round_bf16(rng.standard_normal((B, hw, hw, c)))
    wt = (rng.standard_normal((k, r, r, c)) / np.sqrt(c * r * r)).astype(np.float32)
    pool = session.pool
    xt = autodiff.make_param(pool, x, "x", dtype=BF16)
    wp = autodiff.make_param(pool, wt, "w")
    y = layers.conv2d(xt, wp, st, pad, pool)
    wq = X.round_bf16(wt)
    ref_y = X.round_bf16(X.conv2d_fwd(x, wq, st, pad))
    assert rel(y.data, ref_y) < TOL
    gy = X.round_bf16(rng.standard_normal(y.shape))
    gyt = autodiff.make_data(pool, gy, dtype=BF16)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", y, gyt, pool), pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.gy", gyt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)
    dw_ref = X.conv2d_wgrad(x, gy, wt.shape, st, pad)
    dx_ref = X.round_bf16(X.conv2d_dgrad(gy, wq, x.shape, st, pad))
    assert rel(session.grad_cache.get("w"), dw_ref) < TOL, rel(session.grad_cache.get("w"), dw_ref)
    assert rel(session.grad_cache.get("x"), dx_ref) < TOL, rel(session.grad_cache.get("x"), dx_ref)


def test_stem_at_batch_256(session):
    """The image stem: NCHW float32 host batch -> fused layout change + im2col -> tcgen05 GEMM (K = 27 padded),
    BN statistics, and its weight gradient (the stem has no input gradient)."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16

    rng = np.random.default_rng(7)
    x = rng.standard_normal((B, 3, 32, 32)).astype(np.float32)
    wt = (rng.standard_normal((64, 3, 3, 3)) / np.sqrt(27)).astype(np.float32)
    pool = session.pool
    xt = autodiff.make_data(pool, x)
    wp = autodiff.make_param(pool, wt, "w")
    y = layers.conv2d(xt, wp, 1, 1, pool, layout="nchw")
    xq = X.round_bf16(np.transpose(x, (0, 2, 3, 1)))
    wq = X.round_bf16(wt)
    assert rel(y.data, X.round_bf16(X.conv2d_fwd(xq, wq, 1, 1))) < TOL
    gy = X.round_bf16(rng.standard_normal(y.shape))
    gyt = autodiff.make_data(pool, gy, dtype=BF16)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", y, gyt, pool), pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.gy", gyt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)
    dw_ref = X.conv2d_wgrad(xq, gy, wt.shape, 1, 1)
    assert rel(session.grad_cache.get("w"), dw_ref) < TOL


@pytest.mark.parametrize("acc", [False, True], ids=["single", "accumulated"])
@pytest.mark.parametrize("case", C2_CONVS, ids=_ids)
def test_bn_backward_fused_into_dgrad_at_batch_256(session, case, acc, monkeypatch):
    """BatchNorm(+ReLU) -> conv at the bench batch, where the conv's dgrad completes the gradient of the BatchNorm
    output, so the dgrad epilogue stores it ReLU-masked and emits the BatchNorm-backward channel sums
    (nsk_conv2d_dgrad_bnstats -> nsk_bn_bwd_partials: no reduction pass). ``accumulated``: the BatchNorm output
    has a second consumer whose gradient is already pending (the residual pattern), so the epilogue adds it
    before masking. Checked against the float64 oracle at 1e-3, and against the unfused path (separate
    reduction kernel) to bf16 rounding."""
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16
    from paper_2409_11600_b200.runtime import Session

    hw, k, co, r, st, pad = case  # the BatchNorm has k channels and feeds the conv k -> co
    rng = np.random.default_rng(3000 + sum(case) + acc)
    x = X.round_bf16(rng.standard_normal((B, hw, hw, k)) * 2.0 + 0.3)
    gb = np.stack([rng.uniform(0.5, 1.5, k), rng.uniform(-0.5, 0.5, k)]).astype(np.float32)
    wt = (rng.standard_normal((co, r, r, k)) * np.sqrt(2.0 / (k * r * r))).astype(np.float32)
    p = (hw + 2 * pad - r) // st + 1
    gy = X.round_bf16(rng.standard_normal((B, p, p, co)))
    gy2 = X.round_bf16(rng.standard_normal((B, hw, hw, k)))

    def run(fuse):
        monkeypatch.setattr(layers, "_BNB_FUSE", fuse)
        s = Session(seed=0)
        pool = s.pool
        xt = autodiff.make_param(pool, x, "x", dtype=BF16)
        gbt = autodiff.make_param(pool, gb, "gb")
        wp = autodiff.make_param(pool, wt, "w")
        y = layers.batchnorm(xt, gbt, pool, relu=True)
        tape = s.tape()
        terms = []
        if acc:  # delivered first: the pending gradient the dgrad then accumulates into
            g2 = autodiff.make_data(pool, gy2, dtype=BF16)
            autodiff.push_assignment(tape, "t.gy2", g2)
            terms.append(autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", y, g2, pool), pool))
        out = layers.conv2d(y, wp, st, pad, pool)
        g1 = autodiff.make_data(pool, gy, dtype=BF16)
        autodiff.push_assignment(tape, "t.gy", g1)
        terms.append(autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", out, g1, pool), pool))
        loss = terms[0] if len(terms) == 1 else autodiff.rec_sum_loss(
            autodiff.rec_elementwise("add", terms[0], terms[1], pool), pool)
        y_d = y.data
        autodiff.push_assignment(tape, "t.loss", loss)
        autodiff.backward(tape, s.grad_cache, pool)
        return y_d, s.grad_cache.get("x").astype(np.float64), s.grad_cache.get("gb").astype(np.float64)

    y_d, dx_f, dgb_f = run(True)
    _, dx_u, dgb_u = run(False)
    ref_y, cache = X.batchnorm_fwd(x, gb[0], gb[1], relu=True)
    assert rel(y_d, X.round_bf16(ref_y)) < TOL
    g = X.round_bf16(X.conv2d_dgrad(gy, X.round_bf16(wt), y_d.shape, st, pad))
    if acc:
        g = X.round_bf16(g.astype(np.float64) + gy2)
    dxr, dgr, dbr, _ = X.batchnorm_bwd(g, cache, y_out=y_d, relu=True)
    assert rel(dgb_f, np.stack([dgr, dbr])) < TOL, ("dgamma/dbeta", rel(dgb_f, np.stack([dgr, dbr])))
    assert rel(dx_f, X.round_bf16(dxr)) < TOL, ("dx", rel(dx_f, X.round_bf16(dxr)))
    # fused vs the separate reduction kernel: the same sums in another order
    assert rel(dgb_f, dgb_u) < 1e-4 and rel(dx_f, dx_u) < 1e-3


@pytest.mark.parametrize("case", [c for c in C2_CONVS if c[2] >= 256 and c[3] == 3], ids=_ids)
def test_conv_passes_pair_multicast(session, case, monkeypatch):
    """The opt-in CTA-pair multicast of the filter operand (NSK_MC=1: 2-CTA clusters, each CTA loads half of every
    B stage into both, stages released by both CTAs' MMAs) on the 256-wide layers, split-K included: same bar."""
    test_conv_passes_at_batch_256(session, case, monkeypatch, pair_multicast=True)
