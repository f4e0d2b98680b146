"""Generate golden vectors by running the REAL reference (nsk-mini) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Writes tests/golden/reference_golden.npz. Everything here goes through the
reference's own public API (nsk.tensor, nsk.autodiff, nsk.nn, nsk.dataset);
the resulting arrays pin oracle/ref_ops.py (CPU tests) and the device path
(GPU tests). /root/reference is not needed at test time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
for cand in ("/root/reference/pkg/src", os.path.join(HERE, "..", "..", "baseline", "_ref")):
    if os.path.isdir(os.path.join(cand, "nsk")):
        sys.path.insert(0, cand)
        break

from nsk import autodiff as ad  # noqa: E402
from nsk import nn  # noqa: E402
from nsk.tensor import GradCache, Pool, bias_add, elementwise, matmul_t, onehot, tensor_from_array  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(20260101)
    pool = Pool()

    # matmul_t: 100 random small shapes + a few larger ones
    for i in range(40):
        m, k, n = (int(v) for v in rng.integers(1, 9, size=3))
        x = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        w = rng.uniform(-1, 1, (n, k)).astype(np.float32)
        out[f"mm{i}_x"], out[f"mm{i}_w"] = x, w
        out[f"mm{i}_y"] = matmul_t(tensor_from_array(pool, x), tensor_from_array(pool, w), pool).data.copy()
    x = rng.standard_normal((256, 512)).astype(np.float32)
    w = rng.standard_normal((10, 512)).astype(np.float32)
    out["mmL_x"], out["mmL_w"] = x, w
    out["mmL_y"] = matmul_t(tensor_from_array(pool, x), tensor_from_array(pool, w), pool).data.copy()

    # elementwise kinds
    a = rng.uniform(-4, 4, (17, 23)).astype(np.float32)
    b = rng.uniform(-4, 4, (17, 23)).astype(np.float32)
    out["ew_a"], out["ew_b"] = a, b
    for kind in ("add", "sub", "hadamard", "relu", "sigmoid", "tanh", "neg"):
        bt = tensor_from_array(pool, b) if kind in ("add", "sub", "hadamard") else None
        out[f"ew_{kind}"] = elementwise(kind, tensor_from_array(pool, a), bt, pool).data.copy()
    out["ew_scalar-add"] = elementwise("scalar-add", tensor_from_array(pool, a), 1.25, pool).data.copy()
    out["ew_scalar-mul"] = elementwise("scalar-mul", tensor_from_array(pool, a), -0.75, pool).data.copy()
    bias = rng.uniform(-1, 1, 23).astype(np.float32)
    out["bias"] = bias
    out["bias_add"] = bias_add(tensor_from_array(pool, a), tensor_from_array(pool, bias), pool).data.copy()
    idx = rng.integers(0, 7, 19).astype(np.float32)
    out["oh_idx"] = idx
    out["onehot"] = onehot(tensor_from_array(pool, idx), 7, pool).data.copy()

    # cross-entropy forward + gradient through backward()
    for tag, (m, c) in {"ce10": (32, 10), "ce1000": (16, 1000), "ce2": (8, 2)}.items():
        z = rng.uniform(-5, 5, (m, c)).astype(np.float32)
        t = rng.integers(0, c, m).astype(np.float32)
        cache, tape = GradCache(), ad.Tape()
        zt = ad.make_param(pool, z, "z")
        tt = ad.make_data(pool, t)
        ad.push_assignment(tape, "t", tt)
        loss = ad.rec_cross_entropy(zt, tt, pool)
        ad.push_assignment(tape, "loss", loss)
        lv = loss.item()
        ad.backward(tape, cache, pool)
        out[f"{tag}_z"], out[f"{tag}_t"] = z, t
        out[f"{tag}_loss"] = np.float64(lv)
        out[f"{tag}_grad"] = cache.get("z").copy()

    # hand case x@w + x, sum-loss (test_autodiff.py:87-95)
    cache, tape = GradCache(), ad.Tape()
    xp = ad.make_param(pool, [[2.0]], "x")
    wp = ad.make_param(pool, [[3.0]], "w")
    y = ad.rec_elementwise("add", ad.rec_matmul_t(xp, wp, pool), xp, pool)
    ad.push_assignment(tape, "y", y)
    loss = ad.rec_sum_loss(y, pool)
    ad.push_assignment(tape, "loss", loss)
    ad.backward(tape, cache, pool)
    out["hand_loss"] = np.float64(loss.item())
    out["hand_dx"], out["hand_dw"] = cache.get("x").copy(), cache.get("w").copy()

    # optimizers: SGD-momentum 3 steps, AdamW 10 steps, clip
    shapes = [(5, 7), (11,), (3, 3)]
    ws = [rng.uniform(-1, 1, s).astype(np.float32) for s in shapes]
    gs = [rng.uniform(-1, 1, s).astype(np.float32) for s in shapes]
    for opt in ("sgd", "adamw"):
        group, cache = nn.ParamGroup(), GradCache()
        ts = []
        for i, (w0, g0) in enumerate(zip(ws, gs)):
            t = ad.make_param(pool, w0, f"p{i}")
            group.add(f"p{i}", t)
            cache.accumulate(f"p{i}", tensor_from_array(pool, g0))
            ts.append(t)
        for _ in range(3 if opt == "sgd" else 10):
            if opt == "sgd":
                nn.sgd_step(group, cache, 0.1, 0.9)
            else:
                nn.adamw_step(group, cache, nn.Hyperparams(learning_rate=0.01, weight_decay=0.01))
        for i, t in enumerate(ts):
            out[f"{opt}_w{i}"] = t.data.copy()
    for i, (w0, g0) in enumerate(zip(ws, gs)):
        out[f"opt_w{i}"], out[f"opt_g{i}"] = w0, g0
    cache = GradCache()
    for i, g0 in enumerate(gs):
        cache.accumulate(f"p{i}", tensor_from_array(pool, g0 * 4))
    out["clip_scale"] = np.float64(nn.clip_grad_norm(cache, 2.0))
    for i in range(len(gs)):
        out[f"clip_g{i}"] = cache.get(f"p{i}").copy()

    # xavier init with a session-style seed draw (builtins.py:89-91)
    srng = np.random.default_rng(0)
    seeds = [int(srng.integers(0, 2**31 - 1)) for _ in range(3)]
    out["xavier_seeds"] = np.array(seeds, np.int64)
    for i, (r, c) in enumerate([(16, 27), (10, 512), (64, 576)]):
        out[f"xavier{i}"] = nn.xavier_uniform_init(r, c, seeds[i], pool).data.copy()

    # a small MLP trained 5 steps end to end (linear -> tanh -> linear -> CE -> SGD)
    from nsk.runtime import Session
    import io
    s = Session(seed=3, workers=1, stdout=io.StringIO(), stderr=io.StringIO())
    from nsk.builtins import BUILTINS
    w1 = BUILTINS["xavier_uniform"](s, None, [16.0, 8.0], 1)
    b1 = BUILTINS["param_zeros"](s, None, [16.0], 1)
    w2 = BUILTINS["xavier_uniform"](s, None, [3.0, 16.0], 1)
    b2 = BUILTINS["param_zeros"](s, None, [3.0], 1)
    xs = rng.standard_normal((24, 8)).astype(np.float32)
    ys = rng.integers(0, 3, 24).astype(np.float32)
    out["mlp_x"], out["mlp_y"] = xs, ys
    losses = []
    for step in range(5):
        x = ad.make_data(s.pool, xs)
        yt = ad.make_data(s.pool, ys)
        s.push_named("s.x", x)
        s.push_named("s.y", yt)
        h = BUILTINS["tanh"](s, None, [BUILTINS["linear"](s, None, [x, w1, b1], 1)], 1)
        s.push_named("s.h", h)
        logits = BUILTINS["linear"](s, None, [h, w2, b2], 1)
        s.push_named("s.logits", logits)
        loss = BUILTINS["cross_entropy"](s, None, [logits, yt], 1)
        s.push_named("s.loss", loss)
        losses.append(loss.item())
        BUILTINS["backward"](s, None, [], 1)
        BUILTINS["sgd_step"](s, None, [0.5, 0.9], 1)
        BUILTINS["zero_grad"](s, None, [], 1)
    out["mlp_losses"] = np.array(losses, np.float64)
    for i, (n, t) in enumerate(s.param_group.params):
        out[f"mlp_final_{i}"] = t.data.copy()

    # dataset: seeded per-epoch permutations (dataset.py:93-102)
    from nsk.dataset import DatasetHandle, batch_rows, reset_epoch
    ds = DatasetHandle(features=np.arange(50, dtype=np.float32).reshape(50, 1), labels=np.zeros(50, np.float32),
                       batch_size=8, shuffle=True, seed=7)
    perms = []
    for _ in range(3):
        reset_epoch(ds)
        perms.append(np.concatenate([batch_rows(ds, i)[0][:, 0] for i in range(ds.num_batches())]))
    out["ds_perms"] = np.stack(perms).astype(np.int64)

    # accuracy (argmax, first max wins)
    z = rng.integers(-2, 3, (64, 5)).astype(np.float32)
    lab = rng.integers(0, 5, 64).astype(np.float32)
    out["acc_z"], out["acc_y"] = z, lab
    out["acc"] = np.float64(np.mean(z.argmax(axis=1) == lab.astype(np.int64)))

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
