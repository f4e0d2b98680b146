"""Whole-network ResNet-18 gradients, device vs the bf16-emulating oracle at batch 8 and 64 (one forward/backward
from initialisation): shows the depth amplification that makes whole-network checks use loss / logits / direction
(early-layer gradients differ by ~25% at both batches while every block alone agrees within 1e-2)."""
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from oracle import models as om
from paper_2409_11600_b200 import _lib, autodiff, nn
from paper_2409_11600_b200.models import ResNet18
from paper_2409_11600_b200.runtime import Session
_lib.ctx.init(0)
for b in (8, 64):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((b, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, b).astype(np.float32)
    s = Session(seed=0)
    model = ResNet18(s)
    ref = om.ResNet18Oracle(seed=0)
    pool = s.pool
    logits = model.forward(autodiff.make_data(pool, x))
    dl = logits.data
    loss = nn.cross_entropy(logits, autodiff.make_data(pool, y), pool)
    s.push_named("loss", loss)
    autodiff.backward(s.tape(), s.grad_cache, pool)
    rl, grads, rlog = ref.loss_and_grads(x, y, bf16=True)
    rel = lambda a, b_: float(np.linalg.norm(np.asarray(a, np.float64) - b_) / max(np.linalg.norm(b_), 1e-30))
    errs = [(key, rel(s.grad_cache.get(n), grads[key])) for (n, _t), key in zip(s.param_group.params, ref.order)]
    print("B", b, "loss", loss.item(), rl, "logits", rel(dl, rlog), "max grad err", max(e for _, e in errs))
    print(sorted(errs, key=lambda t: -t[1])[:8])
