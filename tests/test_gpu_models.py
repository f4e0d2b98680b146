"""Whole-step parity: device training steps vs the CPU oracle on identical seeds and inputs."""

import numpy as np
import pytest

from oracle import models as om

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_small_cnn_one_sgd_step_matches_oracle(session):
    """C1: small CNN, one SGD step at batch 32. Every activation (h1, h2, logits), the loss,
    every parameter gradient and every applied update against the bf16-emulating oracle at the north star's
    1e-3 (normwise relative); init bit-identical."""
    from paper_2409_11600_b200 import autodiff, nn
    from paper_2409_11600_b200.models import SmallCNN

    rng = np.random.default_rng(0)
    x = rng.standard_normal((32, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, 32).astype(np.float32)
    model = SmallCNN(session)
    w0 = {n: t.data.copy() for n, t in session.param_group.params}
    ref = om.SmallCNNOracle(seed=0)
    names = ["w1", "b1", "w2", "b2", "fc_w", "fc_b"]
    for (n, _t), key in zip(session.param_group.params, names):
        np.testing.assert_array_equal(w0[n], ref.params[key])  # bit-identical init (seed plumbing)
    acts = {}
    push = session.push_named

    def record(name, t):  # every statement the model pushes: read its value before backward reclaims it
        acts[name.split(".")[-1]] = t.data.copy()
        push(name, t)

    session.push_named = record
    pool = session.pool
    logits = model.forward(autodiff.make_data(pool, x))
    loss = nn.cross_entropy(logits, autodiff.make_data(pool, y), pool)
    push("loss", loss)
    lv = loss.item()
    autodiff.backward(session.tape(), session.grad_cache, pool)
    grads = {n: session.grad_cache.get(n).copy() for n, _t in session.param_group.params}
    nn.sgd_step(session.param_group, session.grad_cache, 0.01, 0.9)
    session.grad_cache.zero_after_step()

    ref_acts = {}
    ref_loss, ref_grads, _ = ref.loss_and_grads(x, y, bf16=True, acts=ref_acts)
    ref.opt.sgd(ref.params, ref_grads, 0.01, 0.9)
    assert abs(lv - ref_loss) <= 1e-3 * abs(ref_loss), (lv, ref_loss)
    for a in ("h1", "h2", "logits"):
        assert _rel(acts[a], ref_acts[a]) < 1e-3, (a, _rel(acts[a], ref_acts[a]))
    for (pname, t), key in zip(session.param_group.params, names):
        assert _rel(grads[pname], ref_grads[key]) < 1e-3, (key, _rel(grads[pname], ref_grads[key]))
        upd = w0[pname].astype(np.float64) - t.data  # the applied update lr * v
        ref_upd = w0[pname].astype(np.float64) - ref.params[key]
        assert _rel(upd, ref_upd) < 1e-3, (key, _rel(upd, ref_upd))


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


def test_side_stream_weight_gradients_are_bit_identical(dev, monkeypatch):
    """Conv weight gradients forked onto the side stream (side.py) vs all on the compute stream: captured
    ResNet-18 steps give bit-identical losses and parameters (same kernels, same order within each stream;
    the deferred releases keep every input alive until the join)."""
    from paper_2409_11600_b200.models import ResNet18
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(5)
    b = 32
    xs = [rng.standard_normal((b, 3, 32, 32)).astype(np.float32) for _ in range(4)]
    ys = [rng.integers(0, 10, b).astype(np.float32) for _ in range(4)]
    out = {}
    for side in ("1", "0"):
        monkeypatch.setenv("NSK_SIDE_WGRAD", side)
        s = Session(seed=0)
        tr = Trainer(s, ResNet18(s), xs[0].shape, 10, optimizer=("sgd", 0.1, 0.9), graph=True, warmup=1)
        losses = [float(tr.step(x, y)) for x, y in zip(xs, ys)]
        out[side] = (losses, [t.data.copy() for _n, t in s.param_group.params])
    assert out["1"][0] == out["0"][0]
    for a, b2 in zip(out["1"][1], out["0"][1]):
        np.testing.assert_array_equal(a, b2)


def test_resnet50_whole_step_matches_oracle(session):
    """C4 architecture at a reduced 64x64 input (grids 32/16/8/4/2 exercise the im2col-mode convs, the 7x7/2
    stem and the 3x3/2 max-pool), one forward/backward vs the bf16-emulating oracle.

    At initialisation this network is chaotic at this size: the oracle's own bf16 and float64 runs differ by
    ~30% in the logits and their early-layer gradients are uncorrelated. So the whole-step bar is the loss
    (2%), logits within the oracle's own bf16-vs-f64 spread, and the head gradients; op-by-op parity along
    the same network is test_resnet50_layer_chain_parity / test_resnet50_block_backward_parity."""
    from paper_2409_11600_b200 import autodiff, nn
    from paper_2409_11600_b200.models import ResNet50

    rng = np.random.default_rng(4)
    b = 4
    x = rng.standard_normal((b, 3, 64, 64)).astype(np.float32)
    y = rng.integers(0, 1000, b).astype(np.float32)
    model = ResNet50(session)
    assert model.num_params() == 25_557_032
    ref = om.ResNet50Oracle(seed=0)
    for (n, t), key in zip(session.param_group.params, ref.order):
        np.testing.assert_array_equal(t.data, ref.params[key])  # bit-identical init (seed plumbing)
    pool = session.pool
    logits = model.forward(autodiff.make_data(pool, x))
    dlogits = logits.data
    loss = nn.cross_entropy(logits, autodiff.make_data(pool, y), pool)
    session.push_named("loss", loss)
    autodiff.backward(session.tape(), session.grad_cache, pool)
    ref_loss, grads, ref_logits = ref.loss_and_grads(x, y, bf16=True)
    _, _, f64_logits = ref.loss_and_grads(x, y, bf16=False)
    spread = _rel(ref_logits, f64_logits)
    assert abs(loss.item() - ref_loss) <= 2e-2 * abs(ref_loss), (loss.item(), ref_loss)
    assert _rel(dlogits, ref_logits) <= max(2 * spread, 3e-2), (_rel(dlogits, ref_logits), spread)
    names = dict(zip(ref.order, (n for n, _t in session.param_group.params)))
    for key in ("fc_w", "fc_b"):
        g = session.grad_cache.get(names[key]).astype(np.float64).ravel()
        r = grads[key].astype(np.float64).ravel()
        assert float(g @ r / (np.linalg.norm(g) * np.linalg.norm(r))) > 0.9, key
    for n, _t in session.param_group.params:
        assert np.all(np.isfinite(session.grad_cache.get(n)))


def _r50_pair(session):
    from paper_2409_11600_b200.models import ResNet50

    model = ResNet50(session)
    ref = om.ResNet50Oracle(seed=0)
    return model, ref, dict(zip(ref.order, (n for n, _t in session.param_group.params)))


def test_resnet50_layer_chain_parity(session):
    """The ResNet-50 forward, each stage fed the device's own input: stem conv, BN and max-pool at the per-op
    1e-3 bar; each bottleneck block (three bf16-stored conv+BN layers in a chain) at 5e-3."""
    from oracle import restated as X
    from paper_2409_11600_b200 import autodiff, layers

    model, ref, _ = _r50_pair(session)
    pool = session.pool
    q = X.round_bf16
    rng = np.random.default_rng(6)
    x = rng.standard_normal((4, 3, 64, 64)).astype(np.float32)
    stem = layers.conv2d(autodiff.make_data(pool, x), model.stem_w, 2, 3, pool, layout="nchw")
    c0 = X.conv2d_fwd(q(np.transpose(x, (0, 2, 3, 1))), q(ref.params["stem_w"]), 2, 3)
    assert _rel(stem.data, q(c0)) < 1e-3
    bn0 = layers.batchnorm(stem, model.stem_bn, pool, relu=True)
    r0, _ = X.batchnorm_fwd(stem.data.astype(np.float64), ref.params["stem_bn"][0], ref.params["stem_bn"][1],
                            relu=True)
    assert _rel(bn0.data, q(r0)) < 1e-3
    h = layers.maxpool(bn0, 3, 2, 1, pool)
    np.testing.assert_array_equal(h.data, q(X.maxpool_fwd(bn0.data, 3, 2, 1)))
    for i in range(len(model.blocks)):
        hin = h.data.astype(np.float64)
        h = model.block(i, h)
        r, _ = ref.block_fwd(i, hin, bf16=True)
        assert _rel(h.data, r) < 5e-3, (i, _rel(h.data, r))


@pytest.mark.parametrize("block", [0, 1, 3, 7, 13])
def test_resnet50_block_backward_parity(session, block):
    """One bottleneck block (projection / identity shortcut, stride 1 / 2, every grid) forward + backward on
    the device's input, loss = sum(out * G): all parameter gradients and the input gradient vs the oracle.
    Six bf16-stored backward ops in a chain (BN backward subtracts means: ill-conditioned): 2e-2."""
    from oracle import restated as X
    from paper_2409_11600_b200 import autodiff
    from paper_2409_11600_b200._lib import BF16

    model, ref, names = _r50_pair(session)
    pool = session.pool
    cin = model.blocks[block]["w1"].shape[3]  # KRSC filters
    hw = {0: 16, 1: 16, 3: 16, 7: 8, 13: 4}[block]
    rng = np.random.default_rng(block)
    hin = X.round_bf16(np.maximum(rng.standard_normal((4, hw, hw, cin)), 0))
    ht = autodiff.make_param(pool, hin, "hin", dtype=BF16)
    out = model.block(block, ht)
    r, cache = ref.block_fwd(block, hin.astype(np.float64), bf16=True)
    assert _rel(out.data, r) < 5e-3
    G = X.round_bf16(rng.standard_normal(out.shape))
    gt = autodiff.make_data(pool, G, dtype=BF16)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", out, gt, pool), pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.g", gt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)
    grads = {}
    dh = ref.block_bwd(G.astype(np.float64), cache, grads, bf16=True)
    errs = {key: _rel(session.grad_cache.get(names[key]), g) for key, g in grads.items()}
    errs["input"] = _rel(session.grad_cache.get("hin"), dh)
    # the oracle's own bf16-vs-float64 spread on the same block, for scale
    _, c64 = ref.block_fwd(block, hin.astype(np.float64), bf16=False)
    g64 = {}
    d64 = ref.block_bwd(G.astype(np.float64), c64, g64, bf16=False)
    spread = {key: _rel(grads[key], g64[key]) for key in grads}
    spread["input"] = _rel(dh, d64)
    print({k: (round(v, 5), round(spread[k], 5)) for k, v in errs.items()})
    for key, e in errs.items():
        assert e < max(2e-2, 2 * spread[key]), (block, key, e, spread[key])


def test_resnet50_graphed_training_steps(dev):
    """ResNet-50 (C4) through the public Trainer with CUDA-graph replay: losses match eager steps."""
    from paper_2409_11600_b200.models import ResNet50
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(5)
    b = 8
    xs = [rng.standard_normal((b, 3, 64, 64)).astype(np.float32) for _ in range(4)]
    ys = [rng.integers(0, 1000, b).astype(np.float32) for _ in range(4)]
    losses = {}
    for mode in (False, True):
        s = Session(seed=0)
        tr = Trainer(s, ResNet50(s), xs[0].shape, 1000, optimizer=("sgd", 0.1, 0.9), graph=mode, warmup=2)
        losses[mode] = [float(tr.step(x, y)) for x, y in zip(xs, ys)]
    np.testing.assert_allclose(losses[True], losses[False], rtol=1e-5)
    assert all(np.isfinite(losses[True]))


@pytest.mark.parametrize("model", ["smallcnn", "resnet18", "resnet18_c2", "resnet18_c2_lr002"])
def test_loss_trajectory_100_steps(dev, model):
    """North star: the loss trajectory stays within 1% of the CPU reference (float64 oracle), on the committed
    golden (tests/golden/gen_trajectory.py: fixed synthetic dataset, reference epoch shuffling, SGD m 0.9; small
    CNN 100 steps at batch 32 and lr 0.01, ResNet-18 30 steps at batch 32 and lr 0.002, and C2 itself: ResNet-18,
    batch 256, lr 0.1, 100 steps over 25,600 rows; and the same at lr 0.02, which does not blow up). Bar: every 10-step window mean within 1% -- or three times
    the oracle's own bf16-vs-float64 window spread in windows where rounding alone moves it by more than 0.5%
    (the lr 0.1 blow-up of C2's first steps). Single steps of a BatchNorm network drift under rounding alone (the
    golden records the oracle's own bf16-emulating run beside the float64 one), so per step: RMS deviation within
    3x the oracle's own bf16-vs-f64 RMS (+0.2%); in the rounding-chaotic windows the worst step within 1.5x the
    oracle's own worst step there, elsewhere no step beyond max(5%, 3x the oracle's own deviation)."""
    import importlib.util
    import os

    from paper_2409_11600_b200.models import ResNet18, SmallCNN
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    spec = importlib.util.spec_from_file_location("gen_trajectory", os.path.join(here, "gen_trajectory.py"))
    G = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(G)
    gold = np.load(os.path.join(here, f"trajectory_{model}.npz"))
    f64, b16 = gold["f64"], gold["bf16"]
    steps, lr, batch, rows_total = G.SETTINGS[model]
    x, y = G.dataset(rows_total)
    sched = G.schedule(len(f64), batch, rows_total)
    s = Session(seed=0)
    net = ResNet18(s) if model.startswith("resnet18") else SmallCNN(s)
    tr = Trainer(s, net, (batch, 3, 32, 32), 10, optimizer=("sgd", lr, G.MOMENTUM), graph=True, warmup=2)
    got = np.array([float(tr.step(x[rows], y[rows])) for rows in sched])
    assert np.all(np.isfinite(got))
    if os.environ.get("NSK_TRAJ_DUMP"):  # diagnostics: the device trajectory
        np.save(os.path.join(os.environ["NSK_TRAJ_DUMP"], f"traj_{model}.npy"), got)
    win = lambda a: a.reshape(-1, 10).mean(axis=1)  # noqa: E731
    rms = lambda a: float(np.sqrt(np.mean(a * a)))  # noqa: E731
    wdev = np.abs(win(got) - win(f64)) / win(f64)
    # 1% per 10-step window; where the oracle's own bf16-emulating run already parts from its float64 run by more
    # than 0.5% (the lr 0.1 blow-up in C2's first 30 steps, loss up to ~13), rounding alone decides the window and
    # the bar is three times that spread
    wspread = np.abs(win(b16) - win(f64)) / win(f64)
    wbar = np.where(wspread > 5e-3, np.maximum(1e-2, 3 * wspread), 1e-2)
    step_dev = np.abs(got - f64) / f64
    spread = np.abs(b16 - f64) / f64
    info = dict(model=model, wdev=np.round(wdev, 4), wbar=np.round(wbar, 4), rms=rms(step_dev), rms_oracle=rms(spread),
                step_max=float(step_dev.max()), step_argmax=int(step_dev.argmax()),
                spread_at=float(spread[step_dev.argmax()]))
    assert np.all(wdev <= wbar), info
    assert rms(step_dev) <= 3 * rms(spread) + 2e-3, info
    # per step: inside the rounding-chaotic windows the worst step within 1.5x the oracle's own worst step there
    # (C2: device 16.6% at step 13, oracle bf16-vs-f64 17.5% at step 17); elsewhere max(5%, 3x the oracle spread)
    chaotic = np.repeat(wspread > 5e-3, 10)
    if chaotic.any():
        assert step_dev[chaotic].max() <= 1.5 * spread[chaotic].max(), info
    calm = ~chaotic
    assert np.all(step_dev[calm] <= np.maximum(5e-2, 3 * spread[calm])), info


def test_step_async_double_buffered_matches_step(dev):
    """Trainer.step_async (copy stream, two input slots, two graphs) reproduces Trainer.step losses."""
    from paper_2409_11600_b200.models import ResNet18
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.train import Trainer

    rng = np.random.default_rng(8)
    b = 16
    xs = [rng.standard_normal((b, 3, 32, 32)).astype(np.float32) for _ in range(7)]
    ys = [rng.integers(0, 10, b).astype(np.float32) for _ in range(7)]
    out = {}
    for mode in ("step", "async"):
        s = Session(seed=0)
        tr = Trainer(s, ResNet18(s), xs[0].shape, 10, optimizer=("sgd", 0.1, 0.9), graph=True, warmup=2)
        fn = tr.step if mode == "step" else tr.step_async
        out[mode] = [float(fn(x, y)) for x, y in zip(xs, ys)]  # a graph's loss slot is reused: read each step
    np.testing.assert_allclose(out["async"], out["step"], rtol=1e-5)


def _r18_block_oracle(ref, pre, st, proj, hin, G, bf16):
    """One ResNet-18 BasicBlock forward + backward composed from the restated ops exactly as ResNet18Oracle does:
    returns (output, {param: gradient}, input gradient)."""
    from oracle import restated as X

    q = X.round_bf16 if bf16 else (lambda a: np.asarray(a, np.float64))
    p = ref.params
    W = {k: q(p[pre + k]) for k in ("w1", "w2") + (("wsc",) if proj else ())}

    def conv_bn(h, wk, bnk, s_, pad, relu, res=None):
        c = q(X.conv2d_fwd(h, W[wk], s_, pad))
        y_, cache = X.batchnorm_fwd(c, p[pre + bnk][0], p[pre + bnk][1], relu=relu, residual=res)
        return q(y_), cache

    o, k1 = conv_bn(hin, "w1", "bn1", st, 1, True)
    sc, ks = conv_bn(hin, "wsc", "bnsc", st, 0, False) if proj else (hin, None)
    h, k2 = conv_bn(o, "w2", "bn2", 1, 1, True, res=sc)
    grads = {}
    dc2, dg, db, dres = X.batchnorm_bwd(G, k2, y_out=h, relu=True)
    dc2, dres = q(dc2), q(dres)
    grads["bn2"] = np.stack([dg, db])
    grads["w2"] = X.conv2d_wgrad(o, dc2, W["w2"].shape, 1, 1)
    do = q(X.conv2d_dgrad(dc2, W["w2"], o.shape, 1, 1))
    dc1, dg, db, _ = X.batchnorm_bwd(do, k1, y_out=o, relu=True)
    dc1 = q(dc1)
    grads["bn1"] = np.stack([dg, db])
    grads["w1"] = X.conv2d_wgrad(hin, dc1, W["w1"].shape, st, 1)
    dhin = q(X.conv2d_dgrad(dc1, W["w1"], hin.shape, st, 1))
    if proj:
        dcs, dg, db, _ = X.batchnorm_bwd(dres, ks, relu=False)
        dcs = q(dcs)
        grads["bnsc"] = np.stack([dg, db])
        grads["wsc"] = X.conv2d_wgrad(hin, dcs, W["wsc"].shape, st, 0)
        dhin = q(dhin + q(X.conv2d_dgrad(dcs, W["wsc"], hin.shape, st, 0)))
    else:
        dhin = q(dhin + dres)
    return h, grads, dhin


@pytest.mark.parametrize("block", [0, 2, 3, 4, 6, 7])
def test_resnet18_block_parity(session, block):
    """C2 block by block (the whole network at initialisation is chaotic under rounding, so each BasicBlock is fed
    the same input on both sides): a ResNet-18 block's forward and every parameter and input gradient through
    the device training path (conv+BN epilogue statistics, fused residual + ReLU, accumulating dgrads, side-stream
    weight gradients) at batch 64, against the bf16-emulating oracle composed like ResNet18Oracle. Bar: 1e-2 for
    the block output and every gradient (a block chains up to six bf16-stored ops; per-op parity is held at 1e-3
    in test_gpu_parity_c2.py). Measured on B200: output 2-7e-4, gradients 2-8e-3 -- while the oracle's own
    bf16-emulating and float64 runs of the same block differ by 4-6 % in the gradients (printed beside)."""
    from oracle import restated as X
    from paper_2409_11600_b200 import autodiff, layers
    from paper_2409_11600_b200._lib import BF16
    from paper_2409_11600_b200.models import ResNet18

    model = ResNet18(session)
    ref = om.ResNet18Oracle(seed=0)
    names = dict(zip(ref.order, (n for n, _t in session.param_group.params)))
    pre, st, proj = ref.blocks[block]
    blk = model.blocks[block]
    cin = blk["w1"].shape[3]
    hw = {0: 32, 2: 32, 3: 16, 4: 16, 6: 8, 7: 8}[block]
    rng = np.random.default_rng(40 + block)
    b = 64
    hin = X.round_bf16(np.maximum(rng.standard_normal((b, hw, hw, cin)), 0))
    pool = session.pool
    ht = autodiff.make_param(pool, hin, "hin", dtype=BF16)
    sc = layers.conv_bn(ht, blk["wsc"], blk["bnsc"], st, 0, pool, relu=False) if "wsc" in blk else ht
    o = layers.conv_bn(ht, blk["w1"], blk["bn1"], st, 1, pool, relu=True)
    out = layers.conv_bn(o, blk["w2"], blk["bn2"], 1, 1, pool, relu=True, residual=sc)
    out_d = out.data
    G = X.round_bf16(rng.standard_normal(out.shape))
    gt = autodiff.make_data(pool, G, dtype=BF16)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", out, gt, pool), pool)
    tape = session.tape()
    autodiff.push_assignment(tape, "t.g", gt)
    autodiff.push_assignment(tape, "t.loss", loss)
    autodiff.backward(tape, session.grad_cache, pool)
    r, grads, dh = _r18_block_oracle(ref, pre, st, proj, hin.astype(np.float64), G.astype(np.float64), True)
    r64, g64, d64 = _r18_block_oracle(ref, pre, st, proj, hin.astype(np.float64), G.astype(np.float64), False)
    errs = {"out": _rel(out_d, r), "input": _rel(session.grad_cache.get("hin"), dh)}
    spread = {"out": _rel(r, r64), "input": _rel(dh, d64)}
    for key, g in grads.items():
        errs[key] = _rel(session.grad_cache.get(names[pre + key]), g)
        spread[key] = _rel(g, g64[key])
    print({k: (round(v, 5), round(spread[k], 5)) for k, v in errs.items()})
    for key, e in errs.items():
        assert e < 1e-2, (block, key, e, spread[key])
