"""Time conv dgrad variants (plain, accumulate, BatchNorm-backward statistics fused) on one geometry.

    python tools/probe_bnstats.py [n hw c k r st pad]      (defaults: the 3x3 64->64 32x32 layer at B=256)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32, ConvDesc  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402

n, hw, c, k, r, st, pad = (int(v) for v in (sys.argv[1:8] if len(sys.argv) > 7 else (256, 32, 64, 64, 3, 1, 1)))
_lib.ctx.init(0)
lib = _lib.lib()
p = (hw + 2 * pad - r) // st + 1
d = ConvDesc(n, hw, hw, c, k, r, r, st, pad, p, p)
rng = np.random.default_rng(0)


def buf(shape, dt=BF16):
    b = Buffer(int(np.prod(shape)), dt)
    b.upload(rng.standard_normal(shape).astype(np.float32))
    return b


dy = buf((n, p, p, k))
w = buf((k, r, r, c))
dx = buf((n, hw, hw, c))
bx = buf((n, hw, hw, c))
mask = Buffer(n * hw * hw * c // 32, F32)
mask.upload(rng.standard_normal(n * hw * hw * c // 32).astype(np.float32))
parts = Buffer(4 * 148 * 2 * c, F32)
s = _lib.stream()
e0, e1 = C.c_void_p(), C.c_void_p()
lib.nsk_event_create(1, C.byref(e0))
lib.nsk_event_create(1, C.byref(e1))
npart = C.c_int(0)


def run(kind):
    if kind == "dgrad":
        return lib.nsk_conv2d_dgrad(C.byref(d), dy.ptr, w.ptr, dx.ptr, s)
    if kind == "dgrad_acc":
        return lib.nsk_conv2d_dgrad_acc(C.byref(d), dy.ptr, w.ptr, dx.ptr, 1.0, s)
    beta = 1.0 if "acc" in kind else 0.0
    mp = None if "nomask" in kind else mask.ptr
    return lib.nsk_conv2d_dgrad_bnstats(C.byref(d), dy.ptr, w.ptr, dx.ptr, beta, bx.ptr, mp, parts.ptr, parts.capacity,
                                        C.byref(npart), s)


KINDS = os.environ.get("KINDS", "dgrad,dgrad_acc,bnstats,bnstats_acc,bnstats_nomask").split(",")
for kind in KINDS:
    for _ in range(3):
        _lib.check(run(kind))
    iters = 20
    lib.nsk_event_record(e0, s)
    for _ in range(iters):
        run(kind)
    lib.nsk_event_record(e1, s)
    lib.nsk_event_sync(e1)
    ms = C.c_float()
    lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
    print(f"{kind:16s} {1000 * ms.value / iters:7.1f} us  (n={n} {hw}x{hw} {c}->{k} {r}x{r} s{st}) probe={os.environ.get('NSK_PROBE', '')}",
          flush=True)
