import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2409_11600_b200 import _lib, autodiff, nn
from paper_2409_11600_b200.models import ResNet18
from paper_2409_11600_b200.runtime import Session
_lib.ctx.init(0)
calls = []
orig_add = autodiff._add_into
def logged(dst, g):
    calls.append(("add_into", dst.shape))
    return orig_add(dst, g)
autodiff._add_into = logged
orig_acc = autodiff._accumulate_slot
def logged2(target, g, pool):
    calls.append(("slot", target.shape, target.grad is None))
    return orig_acc(target, g, pool)
autodiff._accumulate_slot = logged2
s = Session(seed=0); m = ResNet18(s)
rng = np.random.default_rng(0)
x = rng.standard_normal((16,3,32,32)).astype(np.float32); y = rng.integers(0,10,16).astype(np.float32)
logits = m.forward(autodiff.make_data(s.pool, x))
loss = nn.cross_entropy(logits, autodiff.make_data(s.pool, y), s.pool)
s.push_named("loss", loss)
autodiff.backward(s.tape(), s.grad_cache, s.pool)
for c in calls: print(c)
