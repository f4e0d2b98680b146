"""Run BN forward (conv partials path) and backward on a ResNet-18 stage shape a few times, for ncu captures.

    python tools/probe_bn.py [N H W C] [relu] [residual]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib, autodiff, layers  # noqa: E402
from paper_2409_11600_b200._lib import BF16  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402

n, h, w, c = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 32, 32, 64)))
res = len(sys.argv) > 6 and sys.argv[6] == "1"
_lib.ctx.init(0)
s = Session(seed=0)
pool = s.pool
rng = np.random.default_rng(0)
x = autodiff.make_param(pool, rng.standard_normal((n, h, w, c)).astype(np.float32), "x", dtype=BF16)
r = autodiff.make_param(pool, rng.standard_normal((n, h, w, c)).astype(np.float32), "r", dtype=BF16) if res else None
gb = autodiff.make_param(pool, np.stack([np.ones(c), np.zeros(c)]).astype(np.float32), "gb")
g = autodiff.make_data(pool, rng.standard_normal((n, h, w, c)).astype(np.float32), dtype=BF16)
for _ in range(int(os.environ.get("REPS", "3"))):
    y = layers.batchnorm(x, gb, pool, relu=True, residual=r)
    loss = autodiff.rec_sum_loss(autodiff.rec_elementwise("hadamard", y, g, pool), pool)
    t = s.tape()
    autodiff.push_assignment(t, "g", g)
    autodiff.push_assignment(t, "l", loss)
    autodiff.backward(t, s.grad_cache, pool)
_lib.sync()
print("ok")
