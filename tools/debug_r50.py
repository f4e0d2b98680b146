"""Scratch: per-block activation comparison of the device ResNet-50 against the bf16 oracle (64x64 input)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import models as om  # noqa: E402
from oracle import restated as X  # noqa: E402
from paper_2409_11600_b200 import _lib, autodiff, layers  # noqa: E402
from paper_2409_11600_b200.models import ResNet50  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


_lib.ctx.init(0)
hw = int(sys.argv[1]) if len(sys.argv) > 1 else 64
b = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rng = np.random.default_rng(4)
x = rng.standard_normal((b, 3, hw, hw)).astype(np.float32)
s = Session(seed=0)
m = ResNet50(s)
ref = om.ResNet50Oracle(seed=0)
pool = s.pool
q = X.round_bf16
p = ref.params
W = {k: q(v) for k, v in p.items() if v.ndim == 4}
xt = autodiff.make_data(pool, x)
stem = layers.conv2d(xt, m.stem_w, 2, 3, pool, layout="nchw")
xo = q(np.transpose(x, (0, 2, 3, 1)))
c0 = q(X.conv2d_fwd(xo, W["stem_w"], 2, 3))
print("stem conv", rel(stem.data, c0))
bn0 = layers.batchnorm(stem, m.stem_bn, pool, relu=True)
r0, _ = X.batchnorm_fwd(stem.data.astype(np.float64), p["stem_bn"][0], p["stem_bn"][1], relu=True)
print("stem bn (same input)", rel(bn0.data, q(r0)))
mp = layers.maxpool(bn0, 3, 2, 1, pool)
print("maxpool (same input)", rel(mp.data, q(X.maxpool_fwd(bn0.data, 3, 2, 1))))
h = mp
for i, (blk, (pre, st, proj)) in enumerate(zip(m.blocks, ref.blocks)):
    hin = h.data.astype(np.float64)
    o1 = layers.batchnorm(layers.conv2d(h, blk["w1"], 1, 0, pool), blk["bn1"], pool, relu=True)
    c = q(X.conv2d_fwd(hin, W[pre + "w1"], 1, 0))
    r1, _ = X.batchnorm_fwd(c, p[pre + "bn1"][0], p[pre + "bn1"][1], relu=True)
    e1 = rel(o1.data, q(r1))
    c2 = layers.conv2d(o1, blk["w2"], st, 1, pool)
    e2c = rel(c2.data, q(X.conv2d_fwd(o1.data.astype(np.float64), W[pre + "w2"], st, 1)))
    o2 = layers.batchnorm(c2, blk["bn2"], pool, relu=True)
    r2, _ = X.batchnorm_fwd(c2.data.astype(np.float64), p[pre + "bn2"][0], p[pre + "bn2"][1], relu=True)
    e2 = rel(o2.data, q(r2))
    if proj:
        sc = layers.batchnorm(layers.conv2d(h, blk["wsc"], st, 0, pool), blk["bnsc"], pool, relu=False)
    else:
        sc = h
    c3 = layers.conv2d(o2, blk["w3"], 1, 0, pool)
    e3c = rel(c3.data, q(X.conv2d_fwd(o2.data.astype(np.float64), W[pre + "w3"], 1, 0)))
    h = layers.batchnorm(c3, blk["bn3"], pool, relu=True, residual=sc)
    r3, _ = X.batchnorm_fwd(c3.data.astype(np.float64), p[pre + "bn3"][0], p[pre + "bn3"][1], relu=True,
                            residual=sc.data.astype(np.float64))
    print(f"block {i} st{st} {tuple(h.shape)}: bn1 {e1:.2e} conv2 {e2c:.2e} bn2 {e2:.2e} conv3 {e3c:.2e} "
          f"out {rel(h.data, q(r3)):.2e}")
