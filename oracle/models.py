"""CPU oracle training steps for the small CNN (C1), CIFAR ResNet-18 (C2), ImageNet ResNet-50 (C4) and the
GRU classifier (C3). TEST INFRASTRUCTURE ONLY.

Parameters are declared in the same order, with the same names and seed
draws, as paper_2409_11600_b200.models (one ``default_rng(seed).integers(0,
2**31-1)`` per random tensor, builtins.py:89-91), so both sides start from
identical weights. Arithmetic is float64 (ref_ops / restated). With
``bf16=True`` values are rounded to bfloat16 at the points where the device
stores bf16 (activations, their gradients, tensor-core operands), which is
what "the oracle consumes operands rounded to the kernel's input precision"
means for a whole step (SURVEY.md §7 hard part 5).
"""

from __future__ import annotations

import numpy as np

from . import ref_ops as R
from . import restated as X


class _Decl:
    def __init__(self, seed):
        self.rng = np.random.default_rng(seed)
        self.params: dict[str, np.ndarray] = {}
        self.order: list[str] = []
        self.n = 0

    def _name(self, key):
        self.order.append(key)
        self.n += 1
        return key

    def conv(self, key, cout, r, s, cin):
        seed = int(self.rng.integers(0, 2**31 - 1))
        self.params[self._name(key)] = X.xavier_conv(cout, r, s, cin, seed)

    def bn(self, key, c):
        gb = np.zeros((2, c), np.float32)
        gb[0] = 1.0
        self.params[self._name(key)] = gb

    def linear(self, key, rows, cols):
        seed = int(self.rng.integers(0, 2**31 - 1))
        self.params[self._name(key)] = R.xavier_uniform(rows, cols, seed)

    def zeros(self, key, *dims):
        self.params[self._name(key)] = np.zeros(dims, np.float32)


class _Opt:
    """SGD-momentum state per parameter (nn.py:91-99)."""

    def __init__(self, params):
        self.vel = {k: np.zeros_like(v) for k, v in params.items()}

    def sgd(self, params, grads, lr, momentum):
        for k in params:
            params[k], self.vel[k] = R.sgd_update(params[k], grads[k].astype(np.float32), self.vel[k], lr, momentum)


class SmallCNNOracle:
    def __init__(self, seed=0, hw=32, classes=10):
        d = _Decl(seed)
        d.conv("w1", 16, 3, 3, 3)
        d.zeros("b1", 16)
        d.conv("w2", 32, 3, 3, 16)
        d.zeros("b2", 32)
        d.linear("fc_w", classes, 32 * (hw // 2) ** 2)
        d.zeros("fc_b", classes)
        self.params = d.params
        self.opt = _Opt(self.params)

    def loss_and_grads(self, x_nchw, y, bf16=False, acts=None):
        """``acts`` (a dict) receives the activations h1, h2 (NHWC) and the logits."""
        q = X.round_bf16 if bf16 else (lambda a: np.asarray(a, np.float64))
        p = self.params
        x = q(np.transpose(x_nchw, (0, 2, 3, 1)))
        w1, w2 = q(p["w1"]), q(p["w2"])
        c1 = q(X.conv2d_fwd(x, w1, 1, 1))
        a1 = q(c1 + p["b1"])
        h1 = np.maximum(a1, 0)
        c2 = q(X.conv2d_fwd(h1, w2, 2, 1))
        a2 = q(c2 + p["b2"])
        h2 = np.maximum(a2, 0)
        f = h2.reshape(h2.shape[0], -1)
        fcw = q(p["fc_w"]) if bf16 else p["fc_w"].astype(np.float64)
        logits = (f @ fcw.T).astype(np.float32) + p["fc_b"]
        if acts is not None:
            acts.update(h1=h1, h2=h2, logits=logits)
        loss, probs = R.cross_entropy(logits, y)
        g = R.cross_entropy_grad(probs, y).astype(np.float64)
        grads = {"fc_b": g.sum(axis=0)}
        # the device keeps this weight gradient in float32 (10-wide gradient rows are not 16-byte aligned for the
        # bf16 tensor-core path; tensor._matmul) and sums it exactly: no bf16 rounding of g here
        grads["fc_w"] = g.T @ f
        df = q(g @ p["fc_w"].astype(np.float64))
        dh2 = df.reshape(h2.shape)
        da2 = dh2 * (a2 > 0)
        grads["b2"] = da2.reshape(-1, da2.shape[-1]).sum(axis=0)
        grads["w2"] = X.conv2d_wgrad(h1, da2, p["w2"].shape, 2, 1)
        dh1 = q(X.conv2d_dgrad(da2, w2, h1.shape, 2, 1))
        da1 = dh1 * (a1 > 0)
        grads["b1"] = da1.reshape(-1, da1.shape[-1]).sum(axis=0)
        grads["w1"] = X.conv2d_wgrad(x, da1, p["w1"].shape, 1, 1)
        return loss, grads, logits

    def train_step(self, x_nchw, y, lr=0.01, momentum=0.9, bf16=False):
        loss, grads, _ = self.loss_and_grads(x_nchw, y, bf16=bf16)
        self.opt.sgd(self.params, grads, lr, momentum)
        return loss


class ResNet18Oracle:
    """CIFAR ResNet-18 training step (same declaration as paper_2409_11600_b200.models.ResNet18)."""

    STAGES = ((64, 1), (128, 2), (256, 2), (512, 2))

    def __init__(self, seed=0, classes=10):
        d = _Decl(seed)
        d.conv("stem_w", 64, 3, 3, 3)
        d.bn("stem_bn", 64)
        self.blocks = []
        cin = 64
        i = 0
        for cout, stride in self.STAGES:
            for b in range(2):
                st = stride if b == 0 else 1
                pre = f"b{i}_"
                d.conv(pre + "w1", cout, 3, 3, cin)
                d.bn(pre + "bn1", cout)
                d.conv(pre + "w2", cout, 3, 3, cout)
                d.bn(pre + "bn2", cout)
                proj = st != 1 or cin != cout
                if proj:
                    d.conv(pre + "wsc", cout, 1, 1, cin)
                    d.bn(pre + "bnsc", cout)
                self.blocks.append((pre, st, proj))
                cin = cout
                i += 1
        d.linear("fc_w", classes, 512)
        d.zeros("fc_b", classes)
        self.params = d.params
        self.order = d.order
        self.opt = _Opt(self.params)

    def loss_and_grads(self, x_nchw, y, bf16=False):
        q = X.round_bf16 if bf16 else (lambda a: np.asarray(a, np.float64))
        p = self.params
        W = {k: q(v) for k, v in p.items() if v.ndim == 4}
        caches = []

        def conv_bn(h, wk, bnk, st, pad, relu, res=None):
            c = q(X.conv2d_fwd(h, W[wk], st, pad))
            y_, cache = X.batchnorm_fwd(c, p[bnk][0], p[bnk][1], relu=relu, residual=res)
            y_ = q(y_)
            return c, y_, cache

        x = q(np.transpose(x_nchw, (0, 2, 3, 1)))
        c0, h, cache0 = conv_bn(x, "stem_w", "stem_bn", 1, 1, True)
        stem = (x, c0, h, cache0)
        for pre, st, proj in self.blocks:
            hin = h
            c1, o, k1 = conv_bn(hin, pre + "w1", pre + "bn1", st, 1, True)
            if proj:
                cs, sc, ks = conv_bn(hin, pre + "wsc", pre + "bnsc", st, 0, False)
            else:
                cs, sc, ks = None, hin, None
            c2, h, k2 = conv_bn(o, pre + "w2", pre + "bn2", 1, 1, True, res=sc)
            caches.append((pre, st, proj, hin, c1, o, k1, cs, sc, ks, c2, h, k2))
        feat = X.avgpool_fwd(h).astype(np.float32)
        fcw = p["fc_w"]
        logits = R.matmul_t(feat, fcw) + p["fc_b"]
        loss, probs = R.cross_entropy(logits, y)
        g = R.cross_entropy_grad(probs, y)
        grads = {"fc_b": g.astype(np.float64).sum(axis=0), "fc_w": R.plain_matmul(g.T, feat).astype(np.float64)}
        dfeat = R.plain_matmul(g, fcw)
        dh = q(X.avgpool_bwd(dfeat, h.shape))
        for (pre, st, proj, hin, c1, o, k1, cs, sc, ks, c2, hout, k2) in reversed(caches):
            dc2, dg, db, dres = X.batchnorm_bwd(dh, k2, y_out=hout, relu=True)
            dc2, dres = q(dc2), q(dres)
            grads[pre + "bn2"] = np.stack([dg, db])
            grads[pre + "w2"] = X.conv2d_wgrad(o, dc2, W[pre + "w2"].shape, 1, 1)
            do = q(X.conv2d_dgrad(dc2, W[pre + "w2"], o.shape, 1, 1))
            dc1, dg, db, _ = X.batchnorm_bwd(do, k1, y_out=o, relu=True)
            dc1 = q(dc1)
            grads[pre + "bn1"] = np.stack([dg, db])
            grads[pre + "w1"] = X.conv2d_wgrad(hin, dc1, W[pre + "w1"].shape, st, 1)
            dhin = q(X.conv2d_dgrad(dc1, W[pre + "w1"], hin.shape, st, 1))
            if proj:
                dcs, dg, db, _ = X.batchnorm_bwd(dres, ks, relu=False)
                dcs = q(dcs)
                grads[pre + "bnsc"] = np.stack([dg, db])
                grads[pre + "wsc"] = X.conv2d_wgrad(hin, dcs, W[pre + "wsc"].shape, st, 0)
                dhin = q(dhin + q(X.conv2d_dgrad(dcs, W[pre + "wsc"], hin.shape, st, 0)))
            else:
                dhin = q(dhin + dres)
            dh = dhin
        x, c0, h0, cache0 = stem
        dc0, dg, db, _ = X.batchnorm_bwd(dh, cache0, y_out=h0, relu=True)
        dc0 = q(dc0)
        grads["stem_bn"] = np.stack([dg, db])
        grads["stem_w"] = X.conv2d_wgrad(x, dc0, W["stem_w"].shape, 1, 1)
        return loss, grads, logits

    def train_step(self, x_nchw, y, lr=0.1, momentum=0.9, bf16=False):
        loss, grads, _ = self.loss_and_grads(x_nchw, y, bf16=bf16)
        self.opt.sgd(self.params, grads, lr, momentum)
        return loss


class ResNet50Oracle:
    """ImageNet ResNet-50 v1.5 training step (same declaration as paper_2409_11600_b200.models.ResNet50)."""

    STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))

    def __init__(self, seed=0, classes=1000):
        d = _Decl(seed)
        d.conv("stem_w", 64, 7, 7, 3)
        d.bn("stem_bn", 64)
        self.blocks = []
        cin = 64
        i = 0
        for width, nblocks, stride in self.STAGES:
            cout = 4 * width
            for b in range(nblocks):
                st = stride if b == 0 else 1
                pre = f"b{i}_"
                d.conv(pre + "w1", width, 1, 1, cin)
                d.bn(pre + "bn1", width)
                d.conv(pre + "w2", width, 3, 3, width)
                d.bn(pre + "bn2", width)
                d.conv(pre + "w3", cout, 1, 1, width)
                d.bn(pre + "bn3", cout)
                if b == 0:
                    d.conv(pre + "wsc", cout, 1, 1, cin)
                    d.bn(pre + "bnsc", cout)
                self.blocks.append((pre, st, b == 0))
                cin = cout
                i += 1
        d.linear("fc_w", classes, 2048)
        d.zeros("fc_b", classes)
        self.params = d.params
        self.order = d.order
        self.opt = _Opt(self.params)

    def _ops(self, bf16):
        q = X.round_bf16 if bf16 else (lambda a: np.asarray(a, np.float64))
        p = self.params
        W = {k: q(v) for k, v in p.items() if v.ndim == 4}

        def conv_bn(h, wk, bnk, st, pad, relu, res=None):
            c = q(X.conv2d_fwd(h, W[wk], st, pad))
            y_, cache = X.batchnorm_fwd(c, p[bnk][0], p[bnk][1], relu=relu, residual=res)
            return q(y_), cache

        def bn_conv_bwd(dy, cache, y_out, relu, bnk, wk, hin, st, pad, grads, need_dx=True):
            dc, dg, db, dres = X.batchnorm_bwd(dy, cache, y_out=y_out, relu=relu)
            dc = q(dc)
            grads[bnk] = np.stack([dg, db])
            grads[wk] = X.conv2d_wgrad(hin, dc, W[wk].shape, st, pad)
            dx = q(X.conv2d_dgrad(dc, W[wk], hin.shape, st, pad)) if need_dx else None
            return dx, q(dres)

        return q, conv_bn, bn_conv_bwd

    def block_fwd(self, i, hin, bf16=False):
        """Bottleneck block i on input hin (NHWC): returns (output, cache for block_bwd)."""
        q, conv_bn, _ = self._ops(bf16)
        pre, st, proj = self.blocks[i]
        o1, k1 = conv_bn(hin, pre + "w1", pre + "bn1", 1, 0, True)
        o2, k2 = conv_bn(o1, pre + "w2", pre + "bn2", st, 1, True)
        if proj:
            sc, ks = conv_bn(hin, pre + "wsc", pre + "bnsc", st, 0, False)
        else:
            sc, ks = hin, None
        h, k3 = conv_bn(o2, pre + "w3", pre + "bn3", 1, 0, True, res=sc)
        return h, (i, hin, o1, k1, o2, k2, ks, h, k3)

    def block_bwd(self, dh, cache, grads, bf16=False):
        """Gradient of block `cache[0]` w.r.t. its input (parameter gradients into `grads`)."""
        q, _, bn_conv_bwd = self._ops(bf16)
        i, hin, o1, k1, o2, k2, ks, hout, k3 = cache
        pre, st, proj = self.blocks[i]
        do2, dres = bn_conv_bwd(dh, k3, hout, True, pre + "bn3", pre + "w3", o2, 1, 0, grads)
        do1, _ = bn_conv_bwd(do2, k2, o2, True, pre + "bn2", pre + "w2", o1, st, 1, grads)
        dhin, _ = bn_conv_bwd(do1, k1, o1, True, pre + "bn1", pre + "w1", hin, 1, 0, grads)
        if proj:
            dsc, _ = bn_conv_bwd(dres, ks, None, False, pre + "bnsc", pre + "wsc", hin, st, 0, grads)
            return q(dhin + dsc)
        return q(dhin + dres)

    def loss_and_grads(self, x_nchw, y, bf16=False):
        q, conv_bn, bn_conv_bwd = self._ops(bf16)
        p = self.params
        x = q(np.transpose(x_nchw, (0, 2, 3, 1)))
        h0, cache0 = conv_bn(x, "stem_w", "stem_bn", 2, 3, True)
        h = q(X.maxpool_fwd(h0, 3, 2, 1))
        caches = []
        for i in range(len(self.blocks)):
            h, c = self.block_fwd(i, h, bf16)
            caches.append(c)
        feat = X.avgpool_fwd(h).astype(np.float32)
        fcw = p["fc_w"]
        logits = R.matmul_t(feat, fcw) + p["fc_b"]
        loss, probs = R.cross_entropy(logits, y)
        g = R.cross_entropy_grad(probs, y)
        grads = {"fc_b": g.astype(np.float64).sum(axis=0), "fc_w": R.plain_matmul(g.T, feat).astype(np.float64)}
        dh = q(X.avgpool_bwd(R.plain_matmul(g, fcw), h.shape))
        for c in reversed(caches):
            dh = self.block_bwd(dh, c, grads, bf16)
        dh0 = q(X.maxpool_bwd(h0, dh, 3, 2, 1))
        bn_conv_bwd(dh0, cache0, h0, True, "stem_bn", "stem_w", x, 2, 3, grads, need_dx=False)
        return loss, grads, logits

    def train_step(self, x_nchw, y, lr=0.1, momentum=0.9, bf16=False):
        loss, grads, _ = self.loss_and_grads(x_nchw, y, bf16=bf16)
        self.opt.sgd(self.params, grads, lr, momentum)
        return loss


def _sig(z):
    return R.stable_sigmoid(z).astype(np.float64)


class GRUOracle:
    """C3 GRU classifier composed from the reference primitives, float64.

    Same declaration order and seed draws as paper_2409_11600_b200.models.GRUClassifier:
    E = xavier(E, V) (gathered as E^T rows), W_r, W_z, W_n = xavier(H, E), b = 0, U_r, U_z, U_n =
    xavier(H, H), c = 0, head = xavier(classes, H), head bias 0.
    """

    def __init__(self, seed=0, vocab=32768, embed=512, hidden=512, classes=2):
        rng = np.random.default_rng(seed)
        draw = lambda r, c: R.xavier_uniform(r, c, int(rng.integers(0, 2**31 - 1)))  # noqa: E731
        self.H = hidden
        self.params = {"table": np.ascontiguousarray(draw(embed, vocab).T)}
        self.params["w"] = np.concatenate([draw(hidden, embed) for _ in range(3)])
        self.params["b"] = np.zeros(3 * hidden, np.float32)
        self.params["u"] = np.concatenate([draw(hidden, hidden) for _ in range(3)])
        self.params["c"] = np.zeros(3 * hidden, np.float32)
        self.params["head_w"] = draw(classes, hidden)
        self.params["head_b"] = np.zeros(classes, np.float32)
        self.order = ["table", "w", "b", "u", "c", "head_w", "head_b"]

    def loss_and_grads(self, tokens, y, bf16=False, recurrent_bf16=None):
        """float64 composition of the reference primitives. ``bf16=True`` rounds to bfloat16 exactly where the
        device feeds its tensor cores (layers.gru / gru_tc.cu): the embedded inputs and W for the input
        projection, h and U for the recurrent product, dgh for the recurrent backward product, and the operands
        of the batched weight / input gradients (dgx, dgh, x, h_prev, W); the input gradient is stored bf16.
        Gate math, state and accumulation stay float64 (the device: fp32). ``recurrent_bf16=False`` keeps the
        recurrence itself exact (the fp32 cooperative kernel the device uses for shapes the cluster kernel does
        not tile)."""
        q = X.round_bf16 if bf16 else (lambda a: np.asarray(a, np.float64))
        qr = q if (bf16 if recurrent_bf16 is None else recurrent_bf16) else (lambda a: np.asarray(a, np.float64))
        p = {k: v.astype(np.float64) for k, v in self.params.items()}
        H = self.H
        tok = np.asarray(tokens).astype(np.int64)  # [B, T]
        B, T = tok.shape
        W, b, U, c = p["w"], p["b"], p["u"], p["c"]
        Wq, Uq = q(W).astype(np.float64), qr(U).astype(np.float64)
        xs = [q(p["table"][tok[:, t]]).astype(np.float64) for t in range(T)]
        h = np.zeros((B, H))
        cache = []
        for t in range(T):
            gx = xs[t] @ Wq.T + b
            gh = qr(h).astype(np.float64) @ Uq.T + c
            r = _sig(gx[:, :H] + gh[:, :H])
            z = _sig(gx[:, H:2 * H] + gh[:, H:2 * H])
            a = gh[:, 2 * H:]
            n = np.tanh(gx[:, 2 * H:] + r * a)
            hn = n - z * n + z * h
            cache.append((h, r, z, n, a))
            h = hn
        logits = (h @ p["head_w"].T + p["head_b"]).astype(np.float32)
        loss, probs = R.cross_entropy(logits, y)
        g = R.cross_entropy_grad(probs, y).astype(np.float64)
        grads = {"head_b": g.sum(axis=0), "head_w": g.T @ h}
        dh = g @ p["head_w"]
        gW, gU = np.zeros_like(W), np.zeros_like(U)
        gb, gc = np.zeros_like(b), np.zeros_like(c)
        gtable = np.zeros_like(p["table"])
        for t in reversed(range(T)):
            hp, r, z, n, a = cache[t]
            dn = dh * (1 - z)
            dz = dh * (hp - n)
            dnp = dn * (1 - n * n)
            drp = dnp * a * r * (1 - r)
            dzp = dz * z * (1 - z)
            dgx = np.concatenate([drp, dzp, dnp], axis=1)
            dgh = np.concatenate([drp, dzp, dnp * r], axis=1)
            dgxq, dghq = q(dgx).astype(np.float64), q(dgh).astype(np.float64)
            gW += dgxq.T @ xs[t]
            gb += dgx.sum(axis=0)
            gU += dghq.T @ q(hp).astype(np.float64)
            gc += dgh.sum(axis=0)
            np.add.at(gtable, tok[:, t], q(dgxq @ Wq).astype(np.float64))
            dh = dh * z + qr(dgh).astype(np.float64) @ Uq
        grads.update({"w": gW, "b": gb, "u": gU, "c": gc, "table": gtable})
        return loss, grads, logits
