"""Per-step phase timeline of the tcgen05 GRU forward, every CTA, from globaltimer stamps (NSK_GRU_TRACE=1).

Stamps per (CTA, step): 1 / 2 first / last h slice landed (MMA warp), 3 accumulator ready, 5 accumulator tile in
shared memory, 6 gate math done, 7 cluster barrier passed (peers done with h_t), 4 end of the step's work."""
import ctypes as C
import os
import sys

os.environ["NSK_GRU_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2409_11600_b200 import _lib, autodiff  # noqa: E402
from paper_2409_11600_b200.models import GRUClassifier  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402

_lib.ctx.init(0)
lib = _lib.lib()
B, T, H = int(os.environ.get("B", 64)), int(os.environ.get("T", 32)), 512
CL = H // 32
s = Session(seed=0)
m = GRUClassifier(s)
tok = np.random.default_rng(0).integers(0, 32768, (B, T)).astype(np.float32)
for _ in range(3):
    m.forward(autodiff.make_data(s.pool, tok))
    s.tape().clear(s.pool)
buf = np.zeros((CL, T, 16), np.int64)
_lib.check(lib.nsk_gru_trace(buf.ctypes.data, T * CL))
t0 = buf[:, :, 1].min(axis=0)  # per step: earliest first-slice arrival
rel = buf - t0[None, :, None]
order = [1, 2, 3, 5, 6, 7, 4]
names = ["slice0", "sliceN", "acc", "tile", "math", "bar_wait", "step_end"]
print("median over steps 2.., per stamp: min / median / max over CTAs (ns from the step's first wait exit)")
for k, nm in zip(order, names):
    v = np.median(rel[:, 2:, k], axis=1)
    print(f"{nm:7s} {v.min():7.0f} {np.median(v):7.0f} {v.max():7.0f}")
print("step period (ns):", float(np.median(np.diff(t0))))
