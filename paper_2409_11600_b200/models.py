"""Model declarations on the drop-in surface: small CNN (C1), CIFAR ResNet-18 (C2), GRU classifier (C3),
ImageNet ResNet-50 (C4).

Parameters are created through the session exactly like the reference's
``xavier_uniform`` / ``param_zeros`` builtins (builtins.py:85-104): names
``p0, p1, ...`` in declaration order, one ``session.rng`` seed draw per
randomly initialised tensor. oracle/models.py declares the same parameters in
the same order, so both sides start from bit-identical weights.

Forward passes record on the session tape; each block output is pushed as an
assignment, the way the interpreter pushes every statement (runtime.py:192-202).
"""

from __future__ import annotations

import numpy as np

from ._lib import BF16
from .side import SIDE
from . import autodiff, layers, nn
from .runtime import Session
from .tensor import Tensor


class Params:
    """Declaration-order parameter factory bound to a session."""

    def __init__(self, session: Session):
        self.s = session

    def _add(self, t):
        self.s.param_group.add(t.param_name, t)
        return t

    def conv(self, cout, r, s, cin) -> Tensor:
        name = self.s.new_param_name()
        return self._add(nn.xavier_uniform_conv(cout, r, s, cin, self.s.new_seed(), self.s.pool, name))

    def bn(self, c) -> Tensor:
        gb = np.zeros((2, c), np.float32)
        gb[0] = 1.0
        return self._add(autodiff.make_param(self.s.pool, gb, self.s.new_param_name()))

    def linear(self, rows, cols) -> Tensor:
        name = self.s.new_param_name()
        return self._add(nn.xavier_uniform_init(rows, cols, self.s.new_seed(), self.s.pool, name=name))

    def zeros(self, *dims) -> Tensor:
        return self._add(autodiff.make_param(self.s.pool, np.zeros(dims, np.float32), self.s.new_param_name()))


class SmallCNN:
    """C1: conv 3->16 3x3 p1 + b -> ReLU -> conv 16->32 3x3 s2 p1 + b -> ReLU -> flatten (NHWC) -> linear -> CE."""

    def __init__(self, session: Session, hw: int = 32, classes: int = 10):
        P = Params(session)
        self.s = session
        self.w1, self.b1 = P.conv(16, 3, 3, 3), P.zeros(16)
        self.w2, self.b2 = P.conv(32, 3, 3, 16), P.zeros(32)
        feat = 32 * (hw // 2) * (hw // 2)
        self.fc_w, self.fc_b = P.linear(classes, feat), P.zeros(classes)

    def forward(self, x_nchw: Tensor) -> Tensor:
        pool, push = self.s.pool, self.s.push_named
        c1 = layers.conv2d(x_nchw, self.w1, 1, 1, pool, layout="nchw")
        h = autodiff.rec_elementwise("relu", autodiff.rec_bias_add(c1, self.b1, pool), None, pool)
        push("cnn.h1", h)
        h = autodiff.rec_elementwise("relu", autodiff.rec_bias_add(layers.conv2d(h, self.w2, 2, 1, pool), self.b2,
                                                                   pool), None, pool)
        push("cnn.h2", h)
        f = layers.reshape(h, (h.shape[0], h.numel // h.shape[0]), pool)
        logits = nn.linear(f, self.fc_w, self.fc_b, pool)
        push("cnn.logits", logits)
        return logits


class ResNet18:
    """CIFAR ResNet-18: 3x3 stem, no max-pool, [2,2,2,2] BasicBlocks, 1x1 projection shortcuts,
    BN after every conv, global average pool, fc -> 11,173,962 parameters."""

    STAGES = ((64, 1), (128, 2), (256, 2), (512, 2))

    def __init__(self, session: Session, classes: int = 10):
        P = Params(session)
        self.s = session
        self.stem_w, self.stem_bn = P.conv(64, 3, 3, 3), P.bn(64)
        self.blocks = []
        cin = 64
        for cout, stride in self.STAGES:
            for b in range(2):
                st = stride if b == 0 else 1
                blk = {"stride": st, "w1": P.conv(cout, 3, 3, cin), "bn1": P.bn(cout),
                       "w2": P.conv(cout, 3, 3, cout), "bn2": P.bn(cout)}
                if st != 1 or cin != cout:
                    blk["wsc"], blk["bnsc"] = P.conv(cout, 1, 1, cin), P.bn(cout)
                self.blocks.append(blk)
                cin = cout
        self.fc_w, self.fc_b = P.linear(classes, 512), P.zeros(classes)

    def num_params(self) -> int:
        return sum(t.numel for _n, t in self.s.param_group.params)

    def forward(self, x_nchw: Tensor | None = None, x_nhwc: Tensor | None = None, train: bool = True) -> Tensor:
        pool, push = self.s.pool, self.s.push_named
        if x_nhwc is not None:
            stem = layers.conv2d(x_nhwc, self.stem_w, 1, 1, pool)
        else:  # host-layout batch: the NCHW->NHWC change is fused into the stem's im2col gather
            stem = layers.conv2d(x_nchw, self.stem_w, 1, 1, pool, layout="nchw")
        h = layers.batchnorm(stem, self.stem_bn, pool, relu=True, training=train)
        push("rn.stem", h)
        for i, blk in enumerate(self.blocks):
            st = blk["stride"]
            # projection shortcut recorded first: its backward then runs after conv1's and accumulates into dx,
            # which lets the 1x1 stride-2 dgrad skip the three parity classes it has no taps for. Its forward is
            # an independent branch: issued on the side stream, overlapping conv1 (side.py)
            if "wsc" in blk:
                fork = SIDE.enabled()
                if fork:
                    SIDE.branch_begin()
                sc = layers.conv_bn(h, blk["wsc"], blk["bnsc"], st, 0, pool, relu=False, training=train)
                if fork:
                    SIDE.branch_end()
            else:
                sc = h
            o = layers.conv_bn(h, blk["w1"], blk["bn1"], st, 1, pool, relu=True, training=train)
            SIDE.branch_join()
            h = layers.conv_bn(o, blk["w2"], blk["bn2"], 1, 1, pool, relu=True, residual=sc, training=train)
            push(f"rn.block{i}", h)
        feat = layers.avgpool_global(h, pool)
        logits = nn.linear(feat, self.fc_w, self.fc_b, pool)
        push("rn.logits", logits)
        return logits


def resnet18_train_flops_per_image() -> float:
    """Algorithmic training FLOPs per 32x32 image (3.329 GFLOP): forward, wgrad and dgrad
    MACs x 2, without the stem's dgrad (its input needs no gradient)."""
    macs = 0
    h = 32
    stem = h * h * 64 * 27
    macs += stem
    cin = 64
    for cout, stride in ResNet18.STAGES:
        for b in range(2):
            st = stride if b == 0 else 1
            ho = h // st
            macs += ho * ho * cout * cin * 9 + ho * ho * cout * cout * 9
            if st != 1 or cin != cout:
                macs += ho * ho * cout * cin
            h, cin = ho, cout
    macs += 512 * 10
    return 2.0 * (3 * macs - stem)


class ResNet50:
    """ImageNet ResNet-50 (v1.5, stride on the 3x3): 7x7/2 stem, 3x3/2 max-pool, bottleneck stages [3,4,6,3]
    (1x1 reduce, 3x3, 1x1 expand x4, BN after every conv, projection shortcut on each stage's first block),
    global average pool, fc -> 25,557,032 parameters (config C4). Activations NHWC bf16."""

    STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))

    def __init__(self, session: Session, classes: int = 1000):
        P = Params(session)
        self.s = session
        self.stem_w, self.stem_bn = P.conv(64, 7, 7, 3), P.bn(64)
        self.blocks = []
        cin = 64
        for width, nblocks, stride in self.STAGES:
            cout = 4 * width
            for b in range(nblocks):
                st = stride if b == 0 else 1
                blk = {"stride": st, "w1": P.conv(width, 1, 1, cin), "bn1": P.bn(width),
                       "w2": P.conv(width, 3, 3, width), "bn2": P.bn(width),
                       "w3": P.conv(cout, 1, 1, width), "bn3": P.bn(cout)}
                if b == 0:
                    blk["wsc"], blk["bnsc"] = P.conv(cout, 1, 1, cin), P.bn(cout)
                self.blocks.append(blk)
                cin = cout
        self.fc_w, self.fc_b = P.linear(classes, 2048), P.zeros(classes)

    def num_params(self) -> int:
        return sum(t.numel for _n, t in self.s.param_group.params)

    def block(self, i: int, h: Tensor, train: bool = True) -> Tensor:
        """Bottleneck block i: 1x1 reduce -> BN/ReLU -> 3x3 (stride) -> BN/ReLU -> 1x1 expand -> BN (+ shortcut) -> ReLU."""
        pool = self.s.pool
        blk = self.blocks[i]
        st = blk["stride"]
        # projection shortcut first: its (stride-2) dgrad then accumulates into dx last and skips tapless classes.
        # Its forward is an independent branch on the side stream, beside conv1 and conv2 (side.py)
        if "wsc" in blk:
            fork = SIDE.enabled()
            if fork:
                SIDE.branch_begin()
            sc = layers.conv_bn(h, blk["wsc"], blk["bnsc"], st, 0, pool, relu=False, training=train)
            if fork:
                SIDE.branch_end()
        else:
            sc = h
        o = layers.conv_bn(h, blk["w1"], blk["bn1"], 1, 0, pool, relu=True, training=train)
        o = layers.conv_bn(o, blk["w2"], blk["bn2"], st, 1, pool, relu=True, training=train)
        SIDE.branch_join()
        return layers.conv_bn(o, blk["w3"], blk["bn3"], 1, 0, pool, relu=True, residual=sc, training=train)

    def forward(self, x_nchw: Tensor, train: bool = True) -> Tensor:
        pool, push = self.s.pool, self.s.push_named
        stem = layers.conv2d(x_nchw, self.stem_w, 2, 3, pool, layout="nchw")
        h = layers.maxpool(layers.batchnorm(stem, self.stem_bn, pool, relu=True, training=train), 3, 2, 1, pool)
        push("rn.stem", h)
        for i in range(len(self.blocks)):
            h = self.block(i, h, train)
            push(f"rn.block{i}", h)
        feat = layers.avgpool_global(h, pool)
        logits = nn.linear(feat, self.fc_w, self.fc_b, pool)
        push("rn.logits", logits)
        return logits


def resnet50_train_flops_per_image(hw: int = 224, classes: int = 1000) -> float:
    """Algorithmic training FLOPs per image (24.30 GFLOP at 224): forward, wgrad and dgrad
    MACs x 2, without the stem's dgrad."""
    h = (hw + 6 - 7) // 2 + 1
    stem = h * h * 64 * 3 * 49
    h = (h + 2 - 3) // 2 + 1
    macs = stem
    cin = 64
    for width, nblocks, stride in ResNet50.STAGES:
        cout = 4 * width
        for b in range(nblocks):
            st = stride if b == 0 else 1
            ho = (h - 1) // st + 1
            macs += h * h * width * cin + ho * ho * width * width * 9 + ho * ho * cout * width
            if b == 0:
                macs += ho * ho * cout * cin
            h, cin = ho, cout
    macs += 2048 * classes
    return 2.0 * (3 * macs - stem)


class GRUClassifier:
    """C3: token embedding -> fused GRU (h_0 = 0) -> linear head on h_T -> cross-entropy.

    Parameters follow the reference composition: the embedding is onehot(tok) @ E with
    E = xavier_uniform(E, V) (stored transposed as a [V, E] gather table), and each gate has its own
    xavier_uniform(H, E) input weight and xavier_uniform(H, H) recurrent weight (seed draws in the order
    r, z, n), stacked here into W [3H, E] / U [3H, H]; biases b, c start at zero.
    """

    def __init__(self, session: Session, vocab: int = 32768, embed: int = 512, hidden: int = 512,
                 classes: int = 2):
        s = session
        self.s = s
        self.input_classes = vocab  # Trainer validates token ids on the host
        e_vals = nn.xavier_values(embed, vocab, s.new_seed())
        self.table = self._param(np.ascontiguousarray(e_vals.T))
        self.w = self._param(np.concatenate([nn.xavier_values(hidden, embed, s.new_seed()) for _ in range(3)]))
        self.b = self._param(np.zeros(3 * hidden, np.float32))
        self.u = self._param(np.concatenate([nn.xavier_values(hidden, hidden, s.new_seed()) for _ in range(3)]))
        self.c = self._param(np.zeros(3 * hidden, np.float32))
        self.head_w = self._param(nn.xavier_values(classes, hidden, s.new_seed()))
        self.head_b = self._param(np.zeros(classes, np.float32))

    def _param(self, values):
        name = self.s.new_param_name()
        t = autodiff.make_param(self.s.pool, values, name)
        self.s.param_group.add(name, t)
        return t

    def forward(self, tokens: Tensor) -> Tensor:
        pool, push = self.s.pool, self.s.push_named
        steps = tokens.shape[1]
        x = layers.embedding(tokens, self.table, pool, dtype=BF16)  # feeds the bf16 input projection
        push("gru.x", x)
        h = layers.gru(x, self.w, self.b, self.u, self.c, steps, pool)
        push("gru.h", h)
        logits = nn.linear(h, self.head_w, self.head_b, pool)
        push("gru.logits", logits)
        return logits


def gru_train_flops_per_seq(steps: int = 128, embed: int = 512, hidden: int = 512, classes: int = 2) -> float:
    """Dense-GEMM training FLOPs per sequence (1.208 GFLOP at T=128, E=H=512)."""
    fwd = steps * (3 * hidden * embed + 3 * hidden * hidden) + classes * hidden
    return 2.0 * 3 * fwd
