"""Run one conv pass (fprop|dgrad|wgrad) of a ResNet-18 layer a few times, for ncu captures.

    python tools/probe_conv.py fprop 256 32 64 64 3 1 1
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32, ConvDesc  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "fprop"
n, hw, c, k, r, st, pad = (int(v) for v in (sys.argv[2:9] if len(sys.argv) > 8 else (256, 32, 64, 64, 3, 1, 1)))
reps = int(os.environ.get("REPS", "4"))
_lib.ctx.init(0)
lib = _lib.lib()
p = (hw + 2 * pad - r) // st + 1
d = ConvDesc(n, hw, hw, c, k, r, r, st, pad, p, p)
x = Buffer(n * hw * hw * c, BF16)
x.fill(0.25)
w = Buffer(k * r * r * c, BF16)
w.fill(0.01)
y = Buffer(n * p * p * k, BF16)
y.fill(0.5)
dw = Buffer(k * r * r * c, F32)
ws_b = lib.nsk_conv2d_wgrad_workspace(C.byref(d))
ws = Buffer(ws_b // 4 + 1, F32)
s = _lib.stream()
for _ in range(reps):
    if kind == "fprop":
        _lib.check(lib.nsk_conv2d_fprop(C.byref(d), x.ptr, w.ptr, y.ptr, 0, s))
    elif kind == "dgrad":
        _lib.check(lib.nsk_conv2d_dgrad(C.byref(d), y.ptr, w.ptr, x.ptr, s))
    else:
        _lib.check(lib.nsk_conv2d_wgrad(C.byref(d), x.ptr, y.ptr, dw.ptr, 0.0, ws.ptr, ws.nbytes, s))
_lib.sync()
print("ok", kind, n, hw, c, k, r, st, pad)
