"""Per-step phase timeline of the tcgen05 GRU forward (or, with BWD=1, backward), every CTA of the first batch
group, from globaltimer stamps (NSK_GRU_TRACE=1 / 2).

Forward stamps per (CTA, step): 1 / 2 first / last h barrier passed (MMA warp), 3 accumulator ready, 5 accumulator
tile in shared memory, 6 gate math done, 7 cluster barrier passed (peers done with h_t), 4 end of the step's work.
Backward: 0 phase A start (partials of the later step visible), 1 dgh block written, 2 every dgh block in the ring,
3 dgh block landed in shared memory (MMA warp), 4 partial products ready, 5 partials stored."""
import ctypes as C
import os
import sys

BWD = os.environ.get("BWD", "0") == "1"
os.environ["NSK_GRU_TRACE"] = "2" if BWD else "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2409_11600_b200 import _lib, autodiff, nn  # noqa: E402
from paper_2409_11600_b200.models import GRUClassifier  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402

_lib.ctx.init(0)
lib = _lib.lib()
B, T, H = int(os.environ.get("B", 64)), int(os.environ.get("T", 32)), 512
CL = H // 32
s = Session(seed=0)
m = GRUClassifier(s)
tok = np.random.default_rng(0).integers(0, 32768, (B, T)).astype(np.float32)
yl = np.random.default_rng(1).integers(0, 2, B).astype(np.float32)
for _ in range(3):
    logits = m.forward(autodiff.make_data(s.pool, tok))
    if BWD:
        loss = nn.cross_entropy(logits, autodiff.make_data(s.pool, yl), s.pool)
        s.push_named("loss", loss)
        autodiff.backward(s.tape(), s.grad_cache, s.pool)
    s.tape().clear(s.pool)
buf = np.zeros((CL, T, 16), np.int64)
_lib.check(lib.nsk_gru_trace(buf.ctypes.data, T * CL))
if BWD:
    t0 = buf[:, :, 0].min(axis=0)  # per step: earliest phase-A start
    order = [0, 1, 2, 3, 4, 5]
    names = ["A_start", "A_done", "B_start", "dgh_in", "P_ready", "P_store"]
else:
    t0 = buf[:, :, 1].min(axis=0)  # per step: earliest first-slice arrival
    order = [1, 2, 3, 5, 6, 7, 4]
    names = ["slice0", "sliceN", "acc", "tile", "math", "bar_wait", "step_end"]
rel = buf - t0[None, :, None]
print("median over steps 2.., per stamp: min / median / max over CTAs (ns from the step's first wait exit)")
for k, nm in zip(order, names):
    v = np.median(rel[:, 2:, k], axis=1)
    print(f"{nm:7s} {v.min():7.0f} {np.median(v):7.0f} {v.max():7.0f}")
print("step period (ns):", float(np.median(np.diff(t0))))
